# round-1 evidence pass after Gray-order loop walking
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r1r.json 2> gpurun_out/bench_r1r.err || exit 1
for i in 0 3 7; do python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | tail -2; done
for c in c3 c4; do python tools/run_k1.py --config $c --shards 8 --index 5 --reps 4 2>&1 | tail -2; done
for c in c5 c4; do
  ncu --set full --clock-control none --import-source on -k regex:k1_jit -c 1 -f \
    -o gpurun_out/r1_k1_jit_gray_$c python tools/run_k1.py --config $c --reps 1 \
    > gpurun_out/ncu_r_$c.log 2>&1
done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra-configs "" > gpurun_out/b_r.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r1r_launches_bench_c5.csv python bench.py --steps 3 --warmup 3 \
  --no-cpu-baseline --extra-configs "" > gpurun_out/ncu_launch_r.log 2>&1
tail -c 1800 gpurun_out/bench_r1r.json
