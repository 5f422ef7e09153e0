#!/bin/bash
# r2 first GPU pass: new multi-device / robustness tests, the full GPU
# suite, one bench line (with shard emulation and cold start).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/r2a_multi.log 2>&1
echo "multi rc=$?" >> gpurun_out/r2a_multi.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2a_gpu.log 2>&1
echo "suite rc=$?" >> gpurun_out/r2a_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
echo "bench rc=$?" >> gpurun_out/r2a_bench.err
tail -3 gpurun_out/r2a_multi.log gpurun_out/r2a_gpu.log gpurun_out/r2a_bench.err
