"""Supplementary scaling evidence at the size cap (N = 40): the full walk of
a 40-spin lattice and each shard of its 8-way top-bit split, timed on one
GPU through the C ABI (isd_enumerate, device events), with the measured
root tail (K4 gather + K2) of the c5 emulation added: what the P-GPU
efficiency looks like when a shard is 2^37 configurations instead of 2^33.

    python tools/scaling_n40.py [--rows 5 --cols 8] [--tail-us 15.4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1110_2561_b200 as isd  # noqa: E402
from paper_1110_2561_b200.enumeration import enumerate_range_timed  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=int, default=5)
    p.add_argument("--cols", type=int, default=8)
    p.add_argument("--depth", type=int, default=1)
    p.add_argument("--tail-us", type=float, default=15.4,
                   help="root tail per step (K4 + K2 + NVLink allowance)")
    a = p.parse_args()
    spec = isd.LatticeSpec(a.rows, a.cols, a.depth)
    n = spec.num_configs

    def timed(lo, hi):
        best = None
        for _ in range(2):  # the first call tunes the plan of this range
            table, ms = enumerate_range_timed(spec, lo, hi)
            best = ms if best is None else min(best, ms)
        return table, best

    full, full_ms = timed(0, n)
    ok = isd.verify_dos(isd.DoSHistogram(spec, full.view("int64"))).passed
    out = {"lattice": f"{a.rows}x{a.cols}x{a.depth} periodic, N={spec.num_spins}",
           "one_gpu_ms": full_ms, "one_gpu_configs_per_s": n / full_ms * 1e3,
           "verify_dos_passed": ok, "tail_ms": a.tail_us / 1e3}
    for P in (2, 4, 8):
        acc = None
        times = []
        for sh in isd.make_shards(spec, P):
            t, ms = timed(sh.start_index, sh.end_index)
            acc = t.copy() if acc is None else acc + t
            times.append(ms)
        step = max(times) + a.tail_us / 1e3
        out[f"P{P}"] = {"shard_ms": [round(x, 3) for x in times],
                        "projected_step_ms": step,
                        "projected_efficiency": full_ms / (P * step),
                        "combined_tables_exact": bool((acc == full).all())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
