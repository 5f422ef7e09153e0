"""`isingdos` — the reference package's import name, served by the B200
engine (drop-in alias).

    import isingdos            # == paper_1110_2561_b200, under the old name
    from isingdos.oracle import ORACLE_MAX_SPINS, bond_pairs

Each submodule of the reference (/root/reference/pkg/src/isingdos/
{lattice,enumeration,thermo,dosio,bench,cli,oracle}.py) maps to the module
of this package that implements it; `isingdos.oracle` is the cross-check
route (paper_1110_2561_b200.crosscheck).  The submodules are the same module
objects, not copies, so patching `isingdos.bench.full_dos_timed` (as the
reference's tests do, test_bench.py:59) patches what `run_bench` calls.
"""

from paper_1110_2561_b200 import *  # noqa: F401,F403
from paper_1110_2561_b200 import __all__, __version__  # noqa: F401
