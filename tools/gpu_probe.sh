mkdir -p gpurun_out
for ips in 1 4; do
ISD_PROBE=1 ISD_AUTOTUNE=0 ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 3 > gpurun_out/probe4_shard_$ips.log 2>&1
done
ISD_PROBE=1 ISD_AUTOTUNE=0 ISD_BAND_ITEMS_PER_SM=4 python tools/run_k1.py --config c5 --reps 3 > gpurun_out/probe4_full_4.log 2>&1
