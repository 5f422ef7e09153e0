"""`isingdos.oracle` -> paper_1110_2561_b200.crosscheck (the reference's
cross-check names, oracle.py:1-116, on the naive GPU engine)."""
import sys

from paper_1110_2561_b200 import crosscheck as _impl

sys.modules[__name__] = _impl
