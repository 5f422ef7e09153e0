# round-1 pass after dynamic (guided) slot claiming in banded items
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "band or baseline or fuzz" \
  > gpurun_out/gpu_tests_s.log 2>&1; echo "tests exit=$?" >> gpurun_out/gpu_tests_s.log
tail -3 gpurun_out/gpu_tests_s.log
for ips in 1 2; do
  echo "items per SM: $ips"
  ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --reps 6 2>&1 | tail -3
  for i in 0 3; do
    ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | tail -2
  done
done 2>&1 | tee gpurun_out/k1_s.log
ncu --set full --clock-control none --import-source on -k regex:k1_jit -c 1 -f \
  -o gpurun_out/r1_k1_jit_band2_c5 python tools/run_k1.py --config c5 --reps 1 \
  > gpurun_out/ncu_s_c5.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r1s.json 2> gpurun_out/bench_r1s.err
tail -c 1500 gpurun_out/bench_r1s.json
