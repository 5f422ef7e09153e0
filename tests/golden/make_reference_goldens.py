"""Generate golden fixtures by running the reference `isingdos` package itself.

Run in the build container only (the reference is mounted read-only at
/root/reference and does not exist on the GPU box):

    python tests/golden/make_reference_goldens.py small     # seconds
    python tests/golden/make_reference_goldens.py thermo    # seconds
    python tests/golden/make_reference_goldens.py big 6     # ~45 min on 6 cores

Outputs are the reference's own on-disk formats (dosio CSV v1,
/root/reference/pkg/src/isingdos/dosio.py:47-53) and a JSON list of
`ThermoPoint` fields written with repr() so floats round-trip exactly.
Every fixture is produced by the reference's public API
(`full_dos`, `enumerate_shard`, `partition_point`); nothing here is
hand-written data.
"""

import json
import os
import sys
import time

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import isingdos  # the unmodified reference package
    return isingdos


# (rows, cols, depth, coupling) lattices small enough for one core in seconds.
SMALL = [
    (2, 2, 1, 1), (2, 3, 1, 1), (3, 3, 1, 1), (2, 4, 1, 1), (3, 4, 1, 1),
    (4, 3, 1, 1), (4, 4, 1, 1), (2, 2, 2, 1), (2, 2, 3, 1), (3, 3, 2, 1),
    (2, 3, 2, 1), (4, 5, 1, 1), (5, 4, 1, 1), (5, 5, 1, 1), (4, 4, 1, -1),
    (3, 3, 1, -2), (3, 4, 1, 0.5), (2, 2, 2, -1), (3, 5, 1, 1), (6, 4, 1, 1),
    (2, 2, 4, 1), (3, 3, 3, 1),
]

BIG = [(3, 3, 4, 1), (6, 6, 1, 1)]


def name_of(rows, cols, depth, coupling):
    j = str(coupling).replace("-", "m").replace(".", "p")
    return f"dos_{rows}x{cols}x{depth}_J{j}.csv"


def small():
    ref = _ref()
    for rows, cols, depth, j in SMALL:
        spec = ref.LatticeSpec(rows, cols, depth, j)
        dos = ref.full_dos(spec, workers=1)
        assert ref.verify_dos(dos).passed
        ref.write_dos(dos, os.path.join(HERE, name_of(rows, cols, depth, j)))
    # Unaligned tall-column slice (mirrors test_enumeration.py:101-115).
    spec = ref.LatticeSpec(17, 2)
    from isingdos.enumeration import Shard
    part = ref.enumerate_shard(spec, None, Shard(0, 1, 123456, 123456 + 4096))
    cells = part.cells()
    with open(os.path.join(HERE, "slice_17x2_123456_4096.json"), "w") as f:
        json.dump({"rows": 17, "cols": 2, "depth": 1, "coupling": 1,
                   "start": 123456, "end": 123456 + 4096, "cells": cells}, f)
    # Odd shard slices of 5x5 (3-way and 7-way make_shards), for the
    # arbitrary-range path of the kernel.
    spec = ref.LatticeSpec(5, 5)
    out = []
    for p in (3, 7):
        for sh in ref.make_shards(spec, p):
            part = ref.enumerate_shard(spec, ref.build_tables(5), sh)
            out.append({"num_shards": p, "shard_id": sh.shard_id,
                        "start": sh.start_index, "end": sh.end_index,
                        "cells": part.cells()})
    with open(os.path.join(HERE, "shards_5x5.json"), "w") as f:
        json.dump(out, f)


THERMO_CASES = [
    # (rows, cols, depth, J, fields, temperatures)
    (2, 2, 1, 1, [0.0, 0.3], [0.5, 1.0, 2.269, 5.0]),
    (4, 4, 1, 1, [0.0, 0.1, 0.5], [0.5 + 0.05 * i for i in range(91)]),
    (5, 5, 1, 1, [0.0], [0.5 + 0.01 * i for i in range(451)]),
    (4, 4, 1, -1, [0.0, 0.7], [0.3, 1.0, 3.0]),
    (3, 3, 1, -2, [0.0, 1.5], [0.2, 1.1, 4.0]),
    (3, 3, 2, 1, [0.0, 0.1], [1.0 + 0.02 * i for i in range(351)]),
    (3, 4, 1, 0.5, [0.25], [0.05, 0.5, 5.0]),
]


def thermo():
    ref = _ref()
    cases = []
    for rows, cols, depth, j, fields, temps in THERMO_CASES:
        spec = ref.LatticeSpec(rows, cols, depth, j)
        dos = ref.full_dos(spec, workers=1)
        pts = []
        for h in fields:
            for p in ref.thermo_sweep(dos, h, temps):
                pts.append([repr(p.field), repr(p.temperature), repr(p.log_z),
                            repr(p.free_energy), repr(p.internal_energy),
                            repr(p.specific_heat), repr(p.mean_magnetization),
                            repr(p.susceptibility)])
        cases.append({"rows": rows, "cols": cols, "depth": depth,
                      "coupling": j, "dos": name_of(rows, cols, depth, j),
                      "points": pts})
    with open(os.path.join(HERE, "thermo_reference.json"), "w") as f:
        json.dump(cases, f)


def big(workers):
    ref = _ref()
    for rows, cols, depth, j in BIG:
        path = os.path.join(HERE, name_of(rows, cols, depth, j))
        if os.path.exists(path):
            continue
        spec = ref.LatticeSpec(rows, cols, depth, j)
        t0 = time.time()
        dos = ref.full_dos(spec, workers=workers)
        assert ref.verify_dos(dos).passed
        ref.write_dos(dos, path)
        print(f"{path}: {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "small":
        small()
    elif what == "thermo":
        thermo()
    elif what == "big":
        big(int(sys.argv[2]) if len(sys.argv) > 2 else 6)
    else:
        raise SystemExit(f"unknown target {what}")
