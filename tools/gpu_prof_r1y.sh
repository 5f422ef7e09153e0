# per-item phase timing of the banded kernel (ISD_PROBE build: clock64 at
# item start, first chunk, warp end, walk end, flush end)
mkdir -p gpurun_out
for ips in 1 4; do
  ISD_PROBE=1 ISD_AUTOTUNE=0 ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 2 \
    > gpurun_out/probe_shard_$ips.log 2>&1
  ISD_PROBE=1 ISD_AUTOTUNE=0 ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --reps 2 \
    > gpurun_out/probe_full_$ips.log 2>&1
done
grep -c ISDPROBE gpurun_out/probe_*.log
