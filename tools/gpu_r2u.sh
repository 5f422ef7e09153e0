#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_cache.py tests/test_gpu_multi.py -q -m gpu > gpurun_out/r2u_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_tests.log
ISD_BENCH_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --extra-configs "" --no-cold --no-cpu-baseline --no-shard-emulation > gpurun_out/r2u_dist.json 2> gpurun_out/r2u_dist.err; echo "dist rc=$?" >> gpurun_out/r2u_dist.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2u_ref.json 2> gpurun_out/r2u_ref.err; echo "ref rc=$?" >> gpurun_out/r2u_ref.err
tail -3 gpurun_out/r2u_tests.log; tail -1 gpurun_out/r2u_dist.err; tail -c 400 gpurun_out/r2u_dist.json; tail -1 gpurun_out/r2u_ref.err; tail -c 300 gpurun_out/r2u_ref.json
