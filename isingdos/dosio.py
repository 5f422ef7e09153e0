"""`isingdos.dosio` -> paper_1110_2561_b200.dosio (the same module object)."""
import sys

from paper_1110_2561_b200 import dosio as _impl

sys.modules[__name__] = _impl
