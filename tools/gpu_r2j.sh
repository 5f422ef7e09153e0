#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 0 3 7; do timeout 600 python tools/shard_probe.py --index $i; done > gpurun_out/r2j_shard_probe.log 2>&1
timeout 600 python tools/shard_probe.py --shards 1 --index 0 >> gpurun_out/r2j_shard_probe.log 2>&1
cat gpurun_out/r2j_shard_probe.log
