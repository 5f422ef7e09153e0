#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 1 2 3; do ISD_LOOP_BITS=5 timeout 600 python tools/run_k1.py --config c5 --shards 8 --index $i --reps 3; done > gpurun_out/r2n_l5.log 2>&1
cat gpurun_out/r2n_l5.log
