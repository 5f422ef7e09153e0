# full GPU check, then evidence: bench line, launch list, ncu of the c5 walk
# kernel, of one 8-way shard and of K2
mkdir -p gpurun_out
bash tools/gpu_checks.sh > gpurun_out/checks_v.log 2>&1; echo "checks exit=$?" >> gpurun_out/checks_v.log
grep -E "passed|failed|smoke|exit" gpurun_out/checks_v.log
python bench.py > gpurun_out/bench_r1v.json 2> gpurun_out/bench_r1v.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra-configs "" > gpurun_out/b_v.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r1v_launches_bench_c5.csv python bench.py --steps 3 --warmup 3 \
  --no-cpu-baseline --extra-configs "" > gpurun_out/ncu_launch_v.log 2>&1
ISD_AUTOTUNE=0 ncu --set full --clock-control none --import-source on -k regex:k1_jit -c 1 -f \
  -o gpurun_out/r1_k1_jit_band5_c5 python tools/run_k1.py --config c5 --reps 1 \
  > gpurun_out/ncu_v_c5.log 2>&1
ISD_AUTOTUNE=0 ncu --set full --clock-control none --import-source on -k regex:k1_jit -c 1 -f \
  -o gpurun_out/r1_k1_jit_shard8c_c5 python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 1 \
  > gpurun_out/ncu_v_shard.log 2>&1
for i in 0 1 2 3 4 5 6 7; do python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | tail -2 | head -1; done
tail -c 1500 gpurun_out/bench_r1v.json
