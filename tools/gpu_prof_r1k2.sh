# K2 rework (min-H shift, w kept in registers): thermo GPU tests + timing;
# per-shard K1 times of an 8-way split (for the multi-GPU projection)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "thermo or partition or sweep or smoke" \
  > gpurun_out/gpu_tests_k2.log 2>&1; echo "tests exit=$?" >> gpurun_out/gpu_tests_k2.log
tail -2 gpurun_out/gpu_tests_k2.log
for c in c5 c3 c1; do python tools/k2_time.py --config $c 2>&1 | tail -1; done
ncu --set full --clock-control none -k regex:k2_ -c 4 -f -o gpurun_out/r1_k2b_c5 \
  python tools/k2_time.py > gpurun_out/ncu_k2b.log 2>&1
for i in 0 1 2 3 4 5 6 7; do python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | tail -2 | head -1; done
