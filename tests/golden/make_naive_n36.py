"""Second, independent route for the N = 36 goldens the reference cannot
express (BASELINE configs 3 and 4): the C oracle's naive mode (explicit
+/-1 spins, one product per bond — oracle.py:71-91 restated) instead of the
bond-offset masks that produced c3_6x6_free.json / c4_6x6_pmJ_seed1234.json.

    python tests/golden/make_naive_n36.py [threads]     # ~25-30 min each
"""

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import cref, naive  # noqa: E402


def main(threads):
    with open(os.path.join(HERE, "c4_bond_signs.json")) as f:
        signs = json.load(f)["signs"]
    jobs = [("c3_6x6_free_naive.json", 6, 6, 1, 1, False, None),
            ("c4_6x6_pmJ_seed1234_naive.json", 6, 6, 1, 1, True, signs)]
    for name, r, c, d, j, per, sg in jobs:
        path = os.path.join(HERE, name)
        if os.path.exists(path):
            continue
        t0 = time.time()
        t = cref.table(r, c, d, j, per, sg, mode="naive", threads=threads)
        cells = [[int(t[m, e]), m, e] for m in range(t.shape[0])
                 for e in range(t.shape[1]) if t[m, e]]
        with open(path, "w") as f:
            json.dump({"rows": r, "cols": c, "depth": d, "coupling": j,
                       "boundary": "periodic" if per else "free",
                       "signs": sg, "n_spins": r * c * d,
                       "n_bonds": t.shape[1] - 1,
                       "produced_by": "C oracle, naive per-bond mode",
                       "cells_m_idx_e_idx": cells}, f)
        print(f"{name}: {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 6)
