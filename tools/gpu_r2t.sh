#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_tests.log
timeout 600 python tools/e2e_breakdown.py --config c5 > gpurun_out/r2t_e2e.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --extra-configs "" --no-cold --no-cpu-baseline --no-shard-emulation > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
tail -2 gpurun_out/r2t_tests.log; cat gpurun_out/r2t_e2e.log
python -c "
import json; d=json.loads(open('gpurun_out/r2t_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'], d['roofline']['traffic'], d['roofline']['traffic_source'])"
