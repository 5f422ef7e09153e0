"""Estimate shared-memory wavefronts per warp-wide histogram reduction.

For a sample of warp instructions of k1_hoisted (32 lanes = 32 runs whose
indices differ in five run bits, same loop value j and copy c) compute the
bins the lanes hit, map them to words with a candidate layout, and count
wavefronts = max over the 32 banks of distinct words in that bank (lanes on
the same word aggregate for free).  CPU-only design tool.
"""

import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1110_2561_b200.workloads import workloads  # noqa: E402


def bins_of(spec, x):
    m = np.bitwise_count(x).astype(np.int64)
    e = np.zeros_like(m)
    for s, msk, jn in spec.bond_classes():
        e += np.bitwise_count(((x ^ (x >> np.uint64(s))) ^ np.uint64(jn))
                              & np.uint64(msk)).astype(np.int64)
    return m, e


def simulate(spec, k=12, ls=0, layout="dense", warps=400, seed=1, lane_bits=None):
    rng = np.random.default_rng(seed)
    n = spec.num_spins
    runs_total = 1 << (n - k)
    B1 = spec.num_bonds + 1
    total_wf = 0
    count = 0
    for _ in range(warps):
        hi = int(rng.integers(0, runs_total >> 5))
        lanes = np.arange(32, dtype=np.uint64)
        if lane_bits is None:
            r = (((hi >> ls) << (ls + 5)) | (lanes.astype(np.int64) << ls)
                 | (hi & ((1 << ls) - 1))).astype(np.uint64)
        else:
            # lanes scatter into the given run-bit positions
            base = np.uint64(hi)
            r = np.zeros(32, dtype=np.uint64)
            # deposit hi bits into the non-lane positions
            free = [b for b in range(n - k) if b not in lane_bits]
            v = 0
            for i, b in enumerate(free):
                if (hi >> i) & 1:
                    v |= 1 << b
            for L in range(32):
                w = v
                for i, b in enumerate(lane_bits):
                    if (L >> i) & 1:
                        w |= 1 << b
                r[L] = w
        j = int(rng.integers(0, 1 << (k - 5)))
        for c in range(32):
            x = (r << np.uint64(k)) | np.uint64(j << 5) | np.uint64(c)
            m, e = bins_of(spec, x)
            if layout == "dense":
                w = m * B1 + e
            elif layout == "half":  # e parity compressed
                w = m * ((B1 + 1) // 2) + (e >> 1)
            elif layout.startswith("stride"):
                S = int(layout[6:])
                w = m * S + e
            elif layout.startswith("hstride"):
                S = int(layout[7:])
                w = m * S + (e >> 1)
            words = np.unique(w)
            banks = np.bincount(words % 32, minlength=32)
            total_wf += banks.max()
            count += 1
    return total_wf / count


if __name__ == "__main__":
    wl = workloads()
    for name in sys.argv[1:] or ["c5", "c3", "c4"]:
        spec = wl[name].spec
        for layout in ["dense", "half"]:
            for ls in (0, 5, 10, 15):
                print(name, layout, "ls", ls, round(simulate(spec, ls=ls,
                      layout=layout, warps=150), 3), flush=True)


def simulate_rep(spec, k, ls, S, halved, R, skew_words, warps=60, seed=3):
    """Lanes use histogram copy (lane % R) placed skew_words*(lane%R) apart."""
    rng = np.random.default_rng(seed)
    n = spec.num_spins
    run_bits = n - k
    tot = cnt = 0
    lanes = np.arange(32, dtype=np.int64)
    for _ in range(warps):
        hi = int(rng.integers(0, 1 << (run_bits - 5)))
        r = ((hi >> ls) << (ls + 5)) | (lanes << ls) | (hi & ((1 << ls) - 1))
        j = int(rng.integers(0, 1 << (k - 7)))
        for c in rng.integers(0, 128, size=24):
            x = (r.astype(np.uint64) << np.uint64(k)) | np.uint64(j << 7) | np.uint64(c)
            m, e = bins_of(spec, x)
            ep = (e >> 1) if halved else e
            w = m * S + ep + (lanes % R) * skew_words
            words = np.unique(w)
            tot += np.bincount(words % 32, minlength=32).max()
            cnt += 1
    return tot / cnt
