#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 0 1 2; do timeout 600 python tools/shard_probe.py --index $i; done > gpurun_out/r2w_shard_probe.log 2>&1
cat gpurun_out/r2w_shard_probe.log
