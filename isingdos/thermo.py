"""`isingdos.thermo` -> paper_1110_2561_b200.thermo (the same module object)."""
import sys

from paper_1110_2561_b200 import thermo as _impl

sys.modules[__name__] = _impl
