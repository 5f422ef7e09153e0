# separable flush + register unrank + static first chunks: GPU suite, probes
# and the items-per-SM / dynamic-claim sweep
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "band or baseline or full" > gpurun_out/gpu_tests_z.log 2>&1
echo "tests exit=$?" >> gpurun_out/gpu_tests_z.log; tail -2 gpurun_out/gpu_tests_z.log
for ips in 1 4; do
  ISD_PROBE=1 ISD_AUTOTUNE=0 ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 2 \
    > gpurun_out/probe3_shard_$ips.log 2>&1
  ISD_PROBE=1 ISD_AUTOTUNE=0 ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --reps 2 \
    > gpurun_out/probe3_full_$ips.log 2>&1
done
for dyn in 0 1; do for ips in 1 2 4 8; do
  echo "dynamic $dyn items/SM $ips"
  ISD_BAND_DYNAMIC=$dyn ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --reps 4 2>&1 | tail -2 | head -1
  for i in 0 3; do
    ISD_BAND_DYNAMIC=$dyn ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | tail -2 | head -1
  done
done; done 2>&1 | tee gpurun_out/k1_z2.log
