set -x
mkdir -p gpurun_out
for c in c5 c4 c3; do
  python tools/run_k1.py --config $c --reps 3 > gpurun_out/r1p_run_$c.log 2>&1 || exit 1
  ncu --set full --clock-control none --import-source on -k regex:k1_jit -c 1 -f -o gpurun_out/r1_k1_jit_pair_$c python tools/run_k1.py --config $c --reps 1 > gpurun_out/ncu_$c.log 2>&1
done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra-configs "" > gpurun_out/b_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1p_launches_bench_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra-configs "" > gpurun_out/ncu_launch.log 2>&1
ISD_PAIR=0 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_unpaired_c5.json 2>&1
python bench.py --steps 300 --warmup 5 --no-cpu-baseline --extra-configs "" > gpurun_out/bench_sustained300.json 2>&1
tail -c 600 gpurun_out/bench_sustained300.json
