#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_api_semantics.py -q -m gpu -x > gpurun_out/r2l_api.log 2>&1; echo "api rc=$?" >> gpurun_out/r2l_api.log
for i in 0 3; do timeout 600 python tools/shard_probe.py --index $i; done > gpurun_out/r2l_shard_probe.log 2>&1
timeout 600 python tools/shard_probe.py --shards 1 --index 0 >> gpurun_out/r2l_shard_probe.log 2>&1
tail -3 gpurun_out/r2l_api.log; grep -v "^ *[0-9]" gpurun_out/r2l_shard_probe.log
