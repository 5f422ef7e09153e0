# final r1 pass: GPU checks (release + bounds-checked + smoke), bench line,
# a sustained 300-step bench, launch list, ncu of the c5 walk, 8 shards
mkdir -p gpurun_out
bash tools/gpu_checks.sh > gpurun_out/checks_f.log 2>&1; echo "checks exit=$?" >> gpurun_out/checks_f.log
grep -E "passed|failed|smoke|exit" gpurun_out/checks_f.log
python bench.py > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err
python bench.py --steps 300 --warmup 5 --no-cpu-baseline --extra-configs "" > gpurun_out/bench_r1f_sustained300.json 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra-configs "" > gpurun_out/b_f.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r1f_launches_bench_c5.csv python bench.py --steps 3 --warmup 3 \
  --no-cpu-baseline --extra-configs "" > gpurun_out/ncu_launch_f.log 2>&1
ISD_AUTOTUNE=0 ncu --set full --clock-control none --import-source on -k regex:k1_jit -c 1 -f \
  -o gpurun_out/r1_k1_jit_final_c5 python tools/run_k1.py --config c5 --reps 1 \
  > gpurun_out/ncu_f_c5.log 2>&1
for i in 0 1 2 3 4 5 6 7; do python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | grep "rep 3"; done
tail -c 600 gpurun_out/bench_r1f_sustained300.json
