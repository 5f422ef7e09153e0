#!/bin/bash
# r2 pass c: dense K2 (tests, timing, ncu); per-item probes of a 2^33 shard
# and of the full c5 walk; ncu of one shard walk.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "thermo or gather or smoke or sweep or partition or cli" > gpurun_out/r2c_k2tests.log 2>&1
echo "k2 tests rc=$?" >> gpurun_out/r2c_k2tests.log
for c in c1 c2 c3 c4 c5; do timeout 300 python tools/k2_time.py --config $c; done > gpurun_out/r2c_k2time.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k2_ -c 2 -o gpurun_out/r2c_k2 python tools/k2_time.py --config c5 --reps 2 > gpurun_out/r2c_ncu_k2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2c_ncu_k2.log
python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 3 > gpurun_out/r2c_shard3.log 2>&1
ISD_PROBE=1 timeout 300 python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 2 > gpurun_out/r2c_probe_shard3.log 2>&1
ISD_PROBE=1 timeout 300 python tools/run_k1.py --config c5 --reps 2 > gpurun_out/r2c_probe_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k1_jit -s 1 -c 1 -o gpurun_out/r2c_k1_shard3 python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 2 > gpurun_out/r2c_ncu_shard.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2c_ncu_shard.log
tail -2 gpurun_out/r2c_k2tests.log; cat gpurun_out/r2c_k2time.log gpurun_out/r2c_shard3.log; grep -c ISDPROBE gpurun_out/r2c_probe_*.log
