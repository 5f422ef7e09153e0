mkdir -p gpurun_out
bash tools/gpu_checks.sh > gpurun_out/checks_g.log 2>&1; echo "checks exit=$?" >> gpurun_out/checks_g.log
grep -E "passed|failed|smoke|exit" gpurun_out/checks_g.log
python bench.py > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err
python bench.py --steps 300 --warmup 5 --no-cpu-baseline --extra-configs "" > gpurun_out/bench_r1g_sustained300.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r1g_launches_bench_c5.csv python bench.py --steps 3 --warmup 3 \
  --no-cpu-baseline --extra-configs "" > gpurun_out/ncu_launch_g.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_g.json 2>&1
tail -c 900 gpurun_out/bench_r1g.json; tail -c 400 gpurun_out/bench_r1g_sustained300.json; tail -c 400 gpurun_out/bench_ref_g.json
