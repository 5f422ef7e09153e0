"""The reference's vectorised CPU engine, restated in numpy (TEST ONLY).

This is the CPU baseline that bench.py times beside the GPU ("port" in the
`cpu_baseline` record, and the `--impl reference` arm), and a second,
vectorised oracle for lattices too large for the naive loops.

* `classify_words` restates `_classify_batch` (enumeration.py:167-205): per
  column word, popcount and circular-shift LUT gathers when rows <= 16
  (lattice.py:167-190), `np.bitwise_count` otherwise.  Periodic, uniform J
  only — exactly what the reference expresses.
* `classify_masks` is the same walk for free boundaries / per-bond signs:
  unsatisfied bonds counted per bond-offset mask, from the naive oracle's
  own bond list.
* `enumerate_range` restates `enumerate_shard` (enumeration.py:208-235):
  arange batches of DEFAULT_BATCH = 8192 (enumeration.py:27), e_idx mirror
  for J < 0 (232-233), `np.bincount` accumulation (234).
* `partition_point` restates thermo.py:37-88.
"""

import os
import time
from multiprocessing import Pool

import numpy as np

from . import naive

DEFAULT_BATCH = 1 << 13


class Lattice:
    """Geometry of one lattice, built from the naive oracle's bond list."""

    def __init__(self, rows, cols, depth=1, coupling=1, periodic=True,
                 signs=None):
        self.rows, self.cols, self.depth = rows, cols, depth
        self.coupling, self.periodic = coupling, periodic
        self.n = rows * cols * depth
        pairs = naive.bond_pairs(rows, cols, depth, periodic)
        self.b = len(pairs)
        self.signs = list(signs) if signs else None
        self.uniform = periodic and signs is None
        pos = [naive.bit_position(rows, cols, r, c, l)
               for r, c, l in naive.site_order(rows, cols, depth)]
        # group bonds by bit offset; a repeated (i, j) (length-2 axis) opens
        # a second mask so the double bond counts twice
        masks = []
        for k, (i, j) in enumerate(pairs):
            lo, hi = sorted((pos[i], pos[j]))
            d = hi - lo
            neg = ((self.signs[k] if self.signs else 1) * coupling) < 0
            for mk in masks:
                if mk[0] == d and not (mk[1] >> lo) & 1:
                    mk[1] |= 1 << lo
                    if neg:
                        mk[2] |= 1 << lo
                    break
            else:
                masks.append([d, 1 << lo, (1 << lo) if neg else 0])
        self.masks = [(np.uint64(d), np.uint64(m), np.uint64(j))
                      for d, m, j in masks]

    # reference LatticeSpec.word_neighbor_pairs (lattice.py:102-119)
    def word_pairs(self):
        pairs = []
        for layer in range(self.depth):
            base = layer * self.cols
            for c in range(self.cols):
                pairs.append((base + c, base + (c + 1) % self.cols))
        if self.depth > 1:
            for layer in range(self.depth):
                for c in range(self.cols):
                    pairs.append((layer * self.cols + c,
                                  ((layer + 1) % self.depth) * self.cols + c))
        return pairs


def build_tables(rows):
    """popcount / circular-shift LUTs (lattice.py:167-190)."""
    size = 1 << rows
    j = np.arange(size, dtype=np.int64)
    pc = np.bitwise_count(j.astype(np.uint64)).astype(np.int64)
    sh = ((j << 1) | (j >> (rows - 1))) & (size - 1)
    return pc, sh


def classify_words(lat, tables, idx):
    """(ups, anti) per index — enumeration.py:167-205."""
    rows = lat.rows
    nwords = lat.cols * lat.depth
    pairs = lat.word_pairs()
    mask = np.uint64((1 << rows) - 1)
    if tables is not None:
        pc, sh = tables
        words = [((idx >> np.uint64(w * rows)) & mask).astype(np.int64)
                 for w in range(nwords)]
        ups = pc[words[0]].copy()
        anti = pc[words[0] ^ sh[words[0]]].copy()
        for w in words[1:]:
            ups += pc[w]
            anti += pc[w ^ sh[w]]
        for a, b in pairs:
            anti += pc[words[a] ^ words[b]]
    else:
        one, back = np.uint64(1), np.uint64(rows - 1)
        words = [(idx >> np.uint64(w * rows)) & mask for w in range(nwords)]
        ups = np.zeros(idx.shape, dtype=np.int64)
        anti = np.zeros(idx.shape, dtype=np.int64)
        for w in words:
            ups += np.bitwise_count(w).astype(np.int64)
            shifted = ((w << one) | (w >> back)) & mask
            anti += np.bitwise_count(w ^ shifted).astype(np.int64)
        for a, b in pairs:
            anti += np.bitwise_count(words[a] ^ words[b]).astype(np.int64)
    return ups, anti


def classify_masks(lat, idx):
    """(ups, e_idx) per index from bond-offset masks (any boundary/signs)."""
    ups = np.bitwise_count(idx).astype(np.int64)
    e = np.zeros(idx.shape, dtype=np.int64)
    for d, m, j in lat.masks:
        e += np.bitwise_count(((idx ^ (idx >> d)) ^ j) & m).astype(np.int64)
    return ups, e


def enumerate_range(lat, start, end, batch_size=DEFAULT_BATCH):
    """int64 (N+1, B+1) table of [start, end) — enumeration.py:208-235."""
    n, b = lat.n, lat.b
    flat = np.zeros((n + 1) * (b + 1), dtype=np.int64)
    tables = build_tables(lat.rows) if lat.uniform and lat.rows <= 16 else None
    ferro = lat.coupling > 0
    for s in range(start, end, batch_size):
        idx = np.arange(s, min(s + batch_size, end), dtype=np.uint64)
        if lat.uniform:
            ups, anti = classify_words(lat, tables, idx)
            e_idx = anti if ferro else b - anti
        else:
            ups, e_idx = classify_masks(lat, idx)
        flat += np.bincount(ups * (b + 1) + e_idx, minlength=flat.size)
    return flat.reshape(n + 1, b + 1)


def _slice_worker(args):
    lat, start, end = args
    t0 = time.perf_counter()
    table = enumerate_range(lat, start, end)
    return table, time.perf_counter() - t0


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def full_table(lat, procs=None):
    """Whole 2^N walk over a process pool (enumeration.py:365-390)."""
    procs = procs or cores()
    total = 1 << lat.n
    base, extra = divmod(total, procs)
    jobs, s = [], 0
    for i in range(procs):
        size = base + (1 if i < extra else 0)
        jobs.append((lat, s, s + size))
        s += size
    if procs == 1:
        res = [_slice_worker(jobs[0])]
    else:
        with Pool(procs) as pool:
            res = pool.map(_slice_worker, jobs)
    out = res[0][0].copy()
    for t, _ in res[1:]:
        out += t
    return out


def sample_rate(lat, per_proc, procs=None):
    """Configurations/s of the reference algorithm on `procs` host cores.

    Each process walks `per_proc` indices placed at k * 2^N / procs (the
    survey's bounded-sample recipe).  Returns
    (configs_per_s, wall_s, procs).
    """
    procs = procs or cores()
    total = 1 << lat.n
    per_proc = min(per_proc, total // procs)
    jobs = [(lat, k * (total // procs), k * (total // procs) + per_proc)
            for k in range(procs)]
    t0 = time.perf_counter()
    if procs == 1:
        _slice_worker(jobs[0])
    else:
        with Pool(procs) as pool:
            pool.map(_slice_worker, jobs)
    wall = time.perf_counter() - t0
    return procs * per_proc / wall, wall, procs


def partition_point(counts, n, b, scale, h, temperature):
    """thermo.py:37-88 on an int64 table; returns the 7 observables.

    (log_z, free_energy, internal_energy, specific_heat, mean_m, chi,
    mean_abs_m) — the last one is the <|M|> extension.
    """
    m_idx, e_idx = np.nonzero(counts)
    g = counts[m_idx, e_idx].astype(np.float64)
    m = (2 * m_idx - n).astype(np.float64)
    e = (2 * e_idx - b).astype(np.float64) * scale
    energy = e - h * m
    x = -energy / temperature
    shift = x.max()
    w = g * np.exp(x - shift)
    s = w.sum()
    log_z = shift + np.log(s)
    p = w / s
    u = float(p @ energy)
    mean_m = float(p @ m)
    var_e = float(p @ (energy - u) ** 2)
    var_m = float(p @ (m - mean_m) ** 2)
    mean_abs = float(p @ np.abs(m))
    return (float(log_z), float(-temperature * log_z), u,
            var_e / temperature ** 2, mean_m, var_m / temperature, mean_abs)
