# segment-weighted band items: band tests, per-block probe, first-call
# latency, timing sweep
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "band or baseline or full" \
  > gpurun_out/gpu_tests_w5.log 2>&1; echo "tests exit=$?" >> gpurun_out/gpu_tests_w5.log
tail -2 gpurun_out/gpu_tests_w5.log
ISD_PROBE=1 ISD_AUTOTUNE=0 python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 2 > gpurun_out/probe9_shard.log 2>&1
ISD_PROBE=1 ISD_AUTOTUNE=0 python tools/run_k1.py --config c5 --reps 2 > gpurun_out/probe9_full.log 2>&1
for wt in 1 0; do for ips in 1 2 4; do
  echo "weights $wt items/SM $ips"
  ISD_BAND_WEIGHTS=$wt ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --reps 4 2>&1 | grep -E "rep (0|3)" 
  for i in 0 3 7; do
    ISD_BAND_WEIGHTS=$wt ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | tail -2 | head -1
  done
done; done 2>&1 | tee gpurun_out/k1_w5.log
