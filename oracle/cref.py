"""Driver of the C oracle oracle/_ref/enum_ref (TEST ONLY).

The lattice is described from the naive oracle's own geometry
(naive.bond_pairs / naive.bit_position), so the C walk shares no code with
the product package.
"""

import os
import subprocess

import numpy as np

from . import naive

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "_ref", "enum_ref")


def build():
    if not os.path.exists(BIN) or (os.path.getmtime(BIN) <
                                   os.path.getmtime(os.path.join(HERE, "enum_ref.c"))):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return BIN


def bonds(rows, cols, depth=1, coupling=1, periodic=True, signs=None):
    """[(bit_i, bit_j, neg)] in the reference bond order."""
    pos = [naive.bit_position(rows, cols, r, c, l)
           for r, c, l in naive.site_order(rows, cols, depth)]
    pairs = naive.bond_pairs(rows, cols, depth, periodic)
    signs = signs or [1] * len(pairs)
    return [(pos[i], pos[j], int(s * coupling < 0))
            for (i, j), s in zip(pairs, signs)]


def table(rows, cols, depth=1, coupling=1, periodic=True, signs=None,
          mode="mask", threads=None, start=0, end=None):
    """int64 (N+1, B+1) table of [start, end) from the C oracle."""
    build()
    n = rows * cols * depth
    bl = bonds(rows, cols, depth, coupling, periodic, signs)
    end = (1 << n) if end is None else end
    threads = threads or len(os.sched_getaffinity(0))
    text = f"{n} {len(bl)} {1 if mode == 'mask' else 0} {threads} {start} {end}\n"
    text += "".join(f"{i} {j} {g}\n" for i, j, g in bl)
    out = subprocess.run([BIN], input=text, capture_output=True, text=True,
                         check=True).stdout
    vals = np.array([int(v) for v in out.split()], dtype=np.int64)
    return vals.reshape(n + 1, len(bl) + 1)
