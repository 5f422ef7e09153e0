# per-item phase timing of the banded kernel (ISD_PROBE build: thread 0 of
# every block prints clock64 offsets at item start, first chunk, walk end,
# flush stage 1 end and flush end)
mkdir -p gpurun_out
ISD_PROBE=1 ISD_AUTOTUNE=0 python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 2 > gpurun_out/probe5_shard.log 2>&1
ISD_PROBE=1 ISD_AUTOTUNE=0 python tools/run_k1.py --config c5 --reps 2 > gpurun_out/probe5_full.log 2>&1
grep -c ISDPROBE gpurun_out/probe5_*.log
