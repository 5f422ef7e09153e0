"""`isingdos.enumeration` -> paper_1110_2561_b200.enumeration (the same module object)."""
import sys

from paper_1110_2561_b200 import enumeration as _impl

sys.modules[__name__] = _impl
