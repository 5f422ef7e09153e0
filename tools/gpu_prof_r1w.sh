# evidence after the banded-launch changes: bench line, launch list, ncu of
# the c5 walk kernel, of an 8-way shard's kernel and of K2
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r1w.json 2> gpurun_out/bench_r1w.err
tail -c 900 gpurun_out/bench_r1w.json
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra-configs "" > gpurun_out/b_w.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r1w_launches_bench_c5.csv python bench.py --steps 3 --warmup 3 \
  --no-cpu-baseline --extra-configs "" > gpurun_out/ncu_launch_w.log 2>&1
ISD_AUTOTUNE=0 ncu --set full --clock-control none --import-source on -k regex:k1_jit -c 1 -f \
  -o gpurun_out/r1_k1_jit_band3_c5 python tools/run_k1.py --config c5 --reps 1 \
  > gpurun_out/ncu_w_c5.log 2>&1
ISD_AUTOTUNE=0 ncu --set full --clock-control none --import-source on -k regex:k1_jit -c 1 -f \
  -o gpurun_out/r1_k1_jit_shard8_c5 python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 1 \
  > gpurun_out/ncu_w_shard.log 2>&1
ISD_AUTOTUNE=0 python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 4 2>&1 | tail -3
ncu --set full --clock-control none -k regex:k2_ -c 4 -f -o gpurun_out/r1_k2_c5 \
  python tools/k2_time.py > gpurun_out/ncu_w_k2.log 2>&1
python tools/k2_time.py 2>&1 | tail -3
