# dynamic item claims: items-per-SM sweep, full c5 walk and 8-way shards
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider -k "band" \
  > gpurun_out/gpu_tests_x.log 2>&1; echo "tests exit=$?" >> gpurun_out/gpu_tests_x.log
tail -2 gpurun_out/gpu_tests_x.log
for dyn in 1 0; do for ips in 1 2 3 4 6; do
  echo "dynamic $dyn items/SM $ips"
  ISD_BAND_DYNAMIC=$dyn ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --reps 4 2>&1 | tail -2 | head -1
  for i in 0 3; do
    ISD_BAND_DYNAMIC=$dyn ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | tail -2 | head -1
  done
done; done 2>&1 | tee gpurun_out/k1_x.log
