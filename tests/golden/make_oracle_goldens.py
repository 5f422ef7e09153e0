"""Golden tables for the BASELINE lattices the reference cannot express.

BASELINE configs 1 (4x4 free), 3 (6x6 free) and 4 (6x6 periodic, +/-J from
seed 1234) need free boundaries or per-bond signs, which the reference
LatticeSpec lacks (lattice.py:83-85).  Their tables come
from the C oracle (oracle/enum_ref.c, mask formulation), which is itself
pinned against the reference's goldens on every lattice the reference can
express (tests/test_oracle_pins.py).  Config 1 is additionally produced by
the naive per-bond Python oracle and the C naive mode, and all three must
agree.  For cross-checking, the two periodic N=36 lattices the reference
does express (3x3x4 and 6x6) are also walked here.

    python tests/golden/make_oracle_goldens.py [threads]
"""

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle import cref, naive  # noqa: E402

C4_SEED = 1234


def dump(path, rows, cols, depth, coupling, periodic, signs, table, how):
    n, b1 = table.shape
    cells = [[int(table[m, e]), int(m), int(e)]
             for m in range(n) for e in range(b1) if table[m, e]]
    obj = {"rows": rows, "cols": cols, "depth": depth, "coupling": coupling,
           "boundary": "periodic" if periodic else "free",
           "signs": signs, "n_spins": n - 1, "n_bonds": b1 - 1,
           "produced_by": how, "cells_m_idx_e_idx": cells}
    with open(path, "w") as f:
        json.dump(obj, f)


def main(threads):
    nb = len(naive.bond_pairs(6, 6, 1, True))
    signs = naive.random_signs(nb, C4_SEED)
    with open(os.path.join(HERE, "c4_bond_signs.json"), "w") as f:
        json.dump({"rows": 6, "cols": 6, "depth": 1, "boundary": "periodic",
                   "seed": C4_SEED,
                   "rule": "numpy.random.default_rng(seed).random(B) < 0.5 "
                           "-> +1, in oracle.bond_pairs order",
                   "signs": signs}, f)

    # c1: three independent routes must agree
    a = naive.full_dos(4, 4, 1, 1, False)
    b = cref.table(4, 4, 1, 1, False, mode="naive", threads=threads)
    c = cref.table(4, 4, 1, 1, False, mode="mask", threads=threads)
    assert (a == b).all() and (a == c).all()
    dump(os.path.join(HERE, "c1_4x4_free.json"), 4, 4, 1, 1, False, None, c,
         "naive python + C naive + C mask (all equal)")

    jobs = [
        ("c3_6x6_free.json", 6, 6, 1, 1, False, None),
        ("c4_6x6_pmJ_seed1234.json", 6, 6, 1, 1, True, signs),
        ("cx_3x3x4_periodic.json", 3, 3, 4, 1, True, None),
        ("cx_6x6_periodic.json", 6, 6, 1, 1, True, None),
    ]
    for name, r, cc, d, j, per, sg in jobs:
        path = os.path.join(HERE, name)
        if os.path.exists(path):
            continue
        t0 = time.time()
        t = cref.table(r, cc, d, j, per, sg, mode="mask", threads=threads)
        assert int(t.sum()) == 1 << (r * cc * d)
        dump(path, r, cc, d, j, per, sg, t, "C oracle, mask mode")
        print(f"{name}: {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
