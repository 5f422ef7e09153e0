"""Cross-time the autotuned plans of the P shards of a split (c5, P = 8):
shard s walked with the plan tuned for shard j, for every (s, j).

    python tools/shard_cross.py [--config c5] [--shards 8] [--reps 3]

Prints the matrix (ms) and each plan's key fields; writes JSON to
gpurun_out/shard_cross_<config>_P<P>.json.  Shows whether a shard's slower
walk is its plan (another shard's plan is faster on it) or the shard.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_2561_b200 as isd  # noqa: E402
from paper_1110_2561_b200 import _native  # noqa: E402
from paper_1110_2561_b200.enumeration import native_lattice  # noqa: E402
from paper_1110_2561_b200.workloads import workloads  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))  # noqa: E402
import knobs_env  # noqa: E402
knobs_env.apply()


def plan_fields(p):
    return {"fp": _native.plan_fingerprint(p), "pair": p.pair_mode, "l": p.l,
            "band_rows": p.band_rows, "A": p.row_words, "B": p.e_words,
            "P": p.plane_words, "S": list(p.pair_words),
            "lanes": hex(p.lane_mask), "copy": list(p.copy_site),
            "model": round(p.est_wavefronts, 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    spec = workloads()[a.config].spec
    lat = native_lattice(spec)
    shards = isd.make_shards(spec, a.shards)
    plans = []
    for sh in shards:
        _, p = _native.walk_plan(lat, sh.start_index, sh.end_index, 0)
        plans.append(p)

    def t(sh):
        best = 1e30
        for _ in range(a.reps):
            _, ms = _native.enumerate_host(lat, sh.start_index, sh.end_index)
            best = min(best, ms)
        return best

    mat = []
    for j, pj in enumerate(plans):
        row = []
        for sh in shards:
            _native.set_walk_plan(lat, sh.start_index, sh.end_index, pj)
            row.append(t(sh))
        mat.append(row)
        print(f"plan {j}: " + " ".join(f"{x:.4f}" for x in row), flush=True)
    for sh, p in zip(shards, plans):  # restore
        _native.set_walk_plan(lat, sh.start_index, sh.end_index, p)
    own = [mat[s][s] for s in range(len(shards))]
    best = [min(mat[j][s] for j in range(len(plans)))
            for s in range(len(shards))]
    print("own :", " ".join(f"{x:.4f}" for x in own), "max", max(own))
    print("best:", " ".join(f"{x:.4f}" for x in best), "max", max(best))
    for j, p in enumerate(plans):
        print(j, plan_fields(p))
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/shard_cross_{a.config}_P{a.shards}.json", "w") as f:
        json.dump({"ms": mat, "own": own, "best": best,
                   "plans": [plan_fields(p) for p in plans]}, f, indent=1)


if __name__ == "__main__":
    main()
