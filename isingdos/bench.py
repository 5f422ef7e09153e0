"""`isingdos.bench` -> paper_1110_2561_b200.bench (the same module object)."""
import sys

from paper_1110_2561_b200 import bench as _impl

sys.modules[__name__] = _impl
