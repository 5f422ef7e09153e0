"""Per-item cost of a banded launch, measured vs the host model.

    python tools/shard_probe.py [--config c5] [--shards 8] [--index 3]

Tunes (or loads) the plan of the shard, then re-runs it with the ISD_PROBE
kernel build under that same plan (injected with set_walk_plan) and prints,
per popcount class q of the free run bits: the measured SM cycles per slot
(items' walk time / slots, from the probe's clock64 marks) next to the host
model's expected wavefronts per RED (band_costs).  If they disagree, the
cost-weighted item cut cannot balance the blocks.
"""

import argparse
import collections
import os
import re
import statistics as st
import subprocess
import sys
from math import comb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_1110_2561_b200 as isd
from paper_1110_2561_b200 import _native
from paper_1110_2561_b200.enumeration import native_lattice
from paper_1110_2561_b200.workloads import workloads
sys.path.insert(0, sys.argv[1] + "/tools")
import knobs_env
knobs_env.apply()  # (ISD_* variables of the caller: force a plan family)
spec = workloads()[sys.argv[2]].spec
P, idx = int(sys.argv[3]), int(sys.argv[4])
sh = isd.make_shards(spec, P)[idx]
lat = native_lattice(spec)
_, plan = _native.walk_plan(lat, sh.start_index, sh.end_index, 0)
t = [ _native.enumerate_host(lat, sh.start_index, sh.end_index)[1] for _ in range(3)]
print("PLAN", plan.k, plan.l, plan.band_rows, hex(plan.lane_mask), plan.row_words,
      list(plan.pair_words), round(plan.est_wavefronts, 4), "ms", min(t), flush=True)
rb = (sh.end_index - sh.start_index).bit_length() - 1 - plan.k
c = _native.band_costs(lat, plan, sh.start_index >> plan.k, rb, 4096, 256)
print("COSTS", rb, " ".join("%.4f" % x for x in c), flush=True)
_native.set_knob("ISD_PROBE", 1)
_native.set_walk_plan(lat, sh.start_index, sh.end_index, plan)
_native.enumerate_host(lat, sh.start_index, sh.end_index)
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--index", type=int, default=3)
    ap.add_argument("--raw", default="", help="also write the probe lines here")
    a = ap.parse_args()
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, a.config,
                        str(a.shards), str(a.index)], capture_output=True,
                       text=True, timeout=900)
    out = r.stdout
    if a.raw:
        with open(a.raw, "w") as fh:
            fh.write(out)
    if r.returncode:
        print(r.stderr[-2000:])
        return 1
    plan = [l for l in out.splitlines() if l.startswith("PLAN")][0]
    print(plan)
    costs_line = [l for l in out.splitlines() if l.startswith("COSTS")][0].split()
    rb = int(costs_line[1])
    costs = [float(x) for x in costs_line[2:]]
    F = rb - 5
    cum = [0]
    for q in range(F + 1):
        cum.append(cum[-1] + comb(F, q))
    model = collections.defaultdict(list)
    for i, cst in enumerate(costs):
        g = (i + 0.5) * (2 ** F) / len(costs)
        q = next(j for j in range(F + 1) if cum[j + 1] > g)
        model[q].append(cst)
    recs = [{k: int(v) for k, v in re.findall(r"(\w+) (-?\d+)", l[9:])}
            for l in out.splitlines() if l.startswith("ISDPROBE")]
    byq = collections.defaultdict(list)
    for x in recs:
        byq[x["q0"]].append((x["walk"], x["slots"]))
    tot = collections.defaultdict(int)
    for x in recs:
        tot[x["blk"]] += x["flush"]
    vals = list(tot.values())
    blk = [tuple(int(v) for v in re.findall(r"(\d+)", l)[0:3])
           for l in out.splitlines() if l.startswith("ISDBLK")]
    if blk:
        enter = [e for _, e, _ in blk]
        leave = [x for _, _, x in blk]
        span = (max(leave) - min(enter)) / 1e3
        print(f"kernel span (first block entry -> last block exit) "
              f"{span:.1f} us; block entry spread "
              f"{(max(enter) - min(enter)) / 1e3:.1f} us; exit spread "
              f"{(max(leave) - min(leave)) / 1e3:.1f} us; mean block "
              f"{sum(x - e for _, e, x in blk) / len(blk) / 1e3:.1f} us")
    print(f"items {len(recs)}; block cycles mean {st.mean(vals):.0f} "
          f"max/mean {max(vals) / st.mean(vals):.4f} min/mean "
          f"{min(vals) / st.mean(vals):.4f}")
    ph = {k: st.mean(x[k] for x in recs) for k in ("first", "walk", "flush")}
    print(f"item phases (SM cycles, mean): start {ph['first']:.0f}, walk ends "
          f"{ph['walk']:.0f}, flush ends {ph['flush']:.0f} "
          f"(flush {ph['flush'] - ph['walk']:.0f})")
    print(" q  items  slots/item  cyc/slot   model(wavefronts/RED)")
    for q in sorted(byq):
        w = byq[q]
        cps = sum(a for a, _ in w) / sum(b for _, b in w)
        m = st.mean(model[q]) if model.get(q) else float("nan")
        print(f"{q:2d} {len(w):5d} {st.mean(b for _, b in w):10.0f} "
              f"{cps:9.1f} {m:10.4f}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
