#!/bin/bash
# r2y: mode 3 with Gray 5 by default and the unrolled flush: parity, times, probe
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -m gpu -x -n 2 2>&1 | tail -3
ISD_LIBRARY=paper_1110_2561_b200/libisingdos_b200_dbg.so timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q -m gpu -x -k "cluster or band" 2>&1 | tail -3
for c in c5 c3 c4; do
  echo "== $c full"
  timeout 600 python tools/run_k1.py --config $c --reps 4 2>&1 | tail -3
done
for i in 0 3 5; do
echo "== c5 shard $i/8"
timeout 600 python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | tail -3
done
timeout 600 python tools/shard_probe.py --config c5 --shards 8 --index 3 --raw gpurun_out/r2y_probe_shard3_raw.txt > gpurun_out/r2y_probe_shard3.txt 2>&1
tail -22 gpurun_out/r2y_probe_shard3.txt
timeout 600 python tools/shard_probe.py --config c5 --shards 1 --index 0 --raw gpurun_out/r2y_probe_full_raw.txt > gpurun_out/r2y_probe_full.txt 2>&1
tail -32 gpurun_out/r2y_probe_full.txt
