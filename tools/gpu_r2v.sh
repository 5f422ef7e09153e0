#!/bin/bash
# r2v: first GPU run of pair mode 3 (cluster of three): parity, then timing
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q -m gpu -x -k "cluster_walk" > gpurun_out/r2v_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_tests.log
tail -5 gpurun_out/r2v_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "paired_and_unpaired and 3" > gpurun_out/r2v_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_tests2.log
tail -5 gpurun_out/r2v_tests2.log
for g in 2 3 4 5; do
  echo "== c5 pair 3 banded gray $g" 
  ISD_PAIR=3 ISD_BAND=1 ISD_GRAY=$g timeout 600 python tools/run_k1.py --config c5 --reps 4 2>&1 | tail -6
done
echo "== c5 default (autotuned over all modes)"
timeout 600 python tools/run_k1.py --config c5 --reps 4 2>&1 | tail -6
