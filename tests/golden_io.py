"""Readers of the committed golden fixtures (test helper).

DoS CSV files use the reference's version-1 format
(/root/reference/pkg/src/isingdos/dosio.py:47-53); the oracle goldens of
lattices the reference cannot express use a small JSON of
[count, m_idx, e_idx] cells.
"""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_csv_table(name):
    """(rows, cols, depth, J, int64 table) from a reference dosio CSV."""
    with open(os.path.join(GOLDEN, name)) as f:
        lines = f.read().splitlines()
    hdr = dict(tok.split("=") for tok in lines[0][2:].split())
    rows, cols, depth = int(hdr["rows"]), int(hdr["cols"]), int(hdr["depth"])
    j = float(hdr["J"])
    j = int(j) if j.is_integer() else j
    n, b = int(hdr["N"]), int(hdr["B"])
    scale = abs(j)
    t = np.zeros((n + 1, b + 1), dtype=np.int64)
    for ln in lines[2:]:
        if not ln.strip():
            continue
        c, m, e = ln.split(",")
        e = float(e) / scale
        t[(int(m) + n) // 2, (int(round(e)) + b) // 2] = int(c)
    return rows, cols, depth, j, t


def read_json_table(name):
    with open(os.path.join(GOLDEN, name)) as f:
        obj = json.load(f)
    t = np.zeros((obj["n_spins"] + 1, obj["n_bonds"] + 1), dtype=np.int64)
    for c, m, e in obj["cells_m_idx_e_idx"]:
        t[m, e] = c
    return obj, t


def csv_goldens():
    return sorted(f for f in os.listdir(GOLDEN)
                  if f.startswith("dos_") and f.endswith(".csv"))


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)
