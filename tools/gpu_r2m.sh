#!/bin/bash
# banded work items: mirrored rows, slot order, measured calibration —
# parity, then c3/c4/c5 walks and shards with and without, per-item probe
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q -m gpu -x -k "mirrored or banded or cluster" -n 2 2>&1 | tail -2
for o in 0 1; do
  for c in c5 c4 c3; do
  echo "== $c full, calibrate $o"
  ISD_BAND_CALIBRATE=$o timeout 600 python tools/run_k1.py --config $c --reps 4 2>&1 | tail -2 | head -1
  done
  for i in 0 3 5; do
  echo "== c5 shard $i/8, calibrate $o"
  ISD_BAND_CALIBRATE=$o timeout 600 python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | tail -2 | head -1
  done
done
timeout 600 python tools/shard_probe.py --config c5 --shards 1 --index 0 --raw gpurun_out/r2m_probe_full_raw.txt > gpurun_out/r2m_probe_full.txt 2>&1
tail -24 gpurun_out/r2m_probe_full.txt | head -8
