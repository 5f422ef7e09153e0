"""`isingdos.lattice` -> paper_1110_2561_b200.lattice (the same module object)."""
import sys

from paper_1110_2561_b200 import lattice as _impl

sys.modules[__name__] = _impl
