#!/bin/bash
# r2 pass b: K2 rewrite (tests + timing + ncu), cross-timed shard plans.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "thermo or gather or smoke or sweep or partition" > gpurun_out/r2b_k2tests.log 2>&1
echo "k2 tests rc=$?" >> gpurun_out/r2b_k2tests.log
for c in c1 c2 c3 c4 c5; do timeout 300 python tools/k2_time.py --config $c; done > gpurun_out/r2b_k2time.log 2>&1
timeout 900 python tools/shard_cross.py --config c5 --shards 8 > gpurun_out/r2b_shard_cross.log 2>&1
echo "cross rc=$?" >> gpurun_out/r2b_shard_cross.log
timeout 600 ncu --set full --clock-control none -k regex:k2_ -c 4 -o gpurun_out/r2b_k2 python tools/k2_time.py --config c5 --reps 2 > gpurun_out/r2b_ncu_k2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2b_ncu_k2.log
tail -2 gpurun_out/r2b_k2tests.log; cat gpurun_out/r2b_k2time.log; tail -12 gpurun_out/r2b_shard_cross.log
