#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "thermo or gather or smoke or sweep or partition or cli" > gpurun_out/r2q_k2tests.log 2>&1
echo "k2 tests rc=$?" >> gpurun_out/r2q_k2tests.log
for c in c1 c2 c3 c4 c5; do timeout 300 python tools/k2_time.py --config $c; done > gpurun_out/r2q_k2time.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k2_ -c 2 -o gpurun_out/r2q_k2 python tools/k2_time.py --config c5 --reps 2 > gpurun_out/r2q_ncu_k2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2q_ncu_k2.log
tail -2 gpurun_out/r2q_k2tests.log; cat gpurun_out/r2q_k2time.log
