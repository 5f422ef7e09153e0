#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/stage_reference_suite.py --src /nonexistent > /dev/null 2>&1
timeout 1500 python bench.py --steps 10 --warmup 3 --extra-configs "" --no-cold --no-cpu-baseline > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err
timeout 1500 python bench.py --steps 10 --warmup 3 --extra-configs "" --no-cold --no-cpu-baseline --knob ISD_LOOP_BITS=5 > gpurun_out/r2o_bench_l5.json 2> gpurun_out/r2o_bench_l5.err
timeout 1800 python -m pytest tests/test_reference_suite.py -q -m gpu > gpurun_out/r2o_refsuite.log 2>&1; echo "refsuite rc=$?" >> gpurun_out/r2o_refsuite.log
python - <<'PY'
import json
for f in ["gpurun_out/r2o_bench.json","gpurun_out/r2o_bench_l5.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "failed", e); continue
    em=d["extra"]["shard_emulation"]
    print(f, d["ms_per_step"], {k:(round(v["max_shard_ms"],4), round(v["tail_ms"],4), round(v["projected_efficiency"],4), v["combined_tables_exact"]) for k,v in em.items() if k.startswith("P")})
    print("  P8 shards", [round(x,4) for x in em["P8"]["shard_ms"]])
PY
tail -5 gpurun_out/r2o_refsuite.log
