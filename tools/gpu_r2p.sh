#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 10 --warmup 3 --extra-configs "" --no-cold --no-cpu-baseline --knob ISD_CLIMB_STEPS=120 --knob ISD_CLIMB_STARTS=6 --knob ISD_TUNE_BANDED=16 > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
python - <<'PY'
import json
for f in ["gpurun_out/r2s_bench.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "failed", e); continue
    em=d["extra"]["shard_emulation"]
    print(f, d["ms_per_step"], {k:(round(v["max_shard_ms"],4), round(v["tail_ms"],4), round(v["projected_efficiency"],4), v["combined_tables_exact"]) for k,v in em.items() if k.startswith("P")})
    for P in ("P4","P8"):
        print(P, [round(x,4) for x in em[P]["shard_ms"]])
        print("  ", [(p["loop_bits"], p["lane_mask"], p["model_wavefronts_per_red"]) for p in em[P]["shard_plans"]])
PY
