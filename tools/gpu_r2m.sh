#!/bin/bash
# mirrored band items: parity, then c5 full walk and shards with and without
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q -m gpu -x -k "mirrored or banded or cluster" -n 2 2>&1 | tail -2
for m in 0 1; do
  echo "== c5 full, mirror $m"
  ISD_BAND_MIRROR=$m timeout 600 python tools/run_k1.py --config c5 --reps 4 2>&1 | tail -3
  for i in 0 3 5; do
  echo "== c5 shard $i/8, mirror $m"
  ISD_BAND_MIRROR=$m timeout 600 python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | tail -2 | head -1
  done
done
timeout 600 python tools/shard_probe.py --config c5 --shards 1 --index 0 --raw gpurun_out/r2m_probe_full_raw.txt > gpurun_out/r2m_probe_full.txt 2>&1
tail -24 gpurun_out/r2m_probe_full.txt
