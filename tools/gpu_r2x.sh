#!/bin/bash
# r2x: mode 3 — Gray level sweep (full c5 walk and an 8-way shard), the
# capture test, and the per-item probe of a shard
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu -x -k "graph_capture" 2>&1 | tail -3
for g in 2 3 4 5; do
  echo "== c5 full, gray $g"
  ISD_GRAY=$g timeout 600 python tools/run_k1.py --config c5 --reps 4 2>&1 | tail -3
  echo "== c5 shard 3/8, gray $g"
  ISD_GRAY=$g timeout 600 python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 4 2>&1 | tail -3
done
for c in c3 c4; do for g in 2 4; do
  echo "== $c full, gray $g"
  ISD_GRAY=$g timeout 600 python tools/run_k1.py --config $c --reps 4 2>&1 | tail -3
done; done
timeout 600 python tools/shard_probe.py --config c5 --shards 8 --index 3 > gpurun_out/r2x_probe_shard3.txt 2>&1
tail -40 gpurun_out/r2x_probe_shard3.txt
