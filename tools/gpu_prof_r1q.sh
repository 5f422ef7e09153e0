# round-1 profiling pass for pairing mode 2 (c3 / c4) and the bench line
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1q.json 2> gpurun_out/bench_r1q.err || exit 1
for c in c3 c4; do
  python tools/run_k1.py --config $c --reps 3 > gpurun_out/r1q_run_$c.log 2>&1 || exit 1
  ncu --set full --clock-control none --import-source on -k regex:k1_jit -c 1 -f \
    -o gpurun_out/r1_k1_jit_pair2_$c python tools/run_k1.py --config $c --reps 1 \
    > gpurun_out/ncu_q_$c.log 2>&1
done
tail -c 2500 gpurun_out/bench_r1q.json
