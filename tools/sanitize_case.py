"""Small workload for compute-sanitizer runs (memcheck / racecheck).

Exercises k1_hoisted (aligned body), k1_canonical (head/tail and tiny
lattices), k3_mirror and k2_thermo on small lattices; checks results.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_2561_b200 as isd  # noqa: E402
from paper_1110_2561_b200 import _native  # noqa: E402
from paper_1110_2561_b200.enumeration import enumerate_range_timed  # noqa: E402

spec = isd.LatticeSpec(4, 5)
full, _ = enumerate_range_timed(spec, 0, spec.num_configs)
part = sum(enumerate_range_timed(spec, a, b)[0]
           for a, b in ((0, 12345), (12345, 700001), (700001, 1 << 20)))
assert np.array_equal(full, part)
flip, _ = enumerate_range_timed(spec, 0, spec.num_configs,
                                algo=_native.FLAG_FLIP_SYMMETRY)
assert np.array_equal(full, flip)
canon, _ = enumerate_range_timed(spec, 0, spec.num_configs,
                                 algo=_native.ALGO_CANONICAL)
assert np.array_equal(full, canon)
signed = isd.LatticeSpec(3, 3, 2, bond_signs=isd.random_bond_signs(
    isd.LatticeSpec(3, 3, 2), 7))
t2, _ = enumerate_range_timed(signed, 0, signed.num_configs)
dos = isd.DoSHistogram(spec, full.view(np.int64))
assert isd.verify_dos(dos).passed
pts = isd.thermo_sweep(dos, 0.1, [0.5, 1.0, 2.0])
print("sanitize case ok", pts[0].log_z, int(t2.sum()))
