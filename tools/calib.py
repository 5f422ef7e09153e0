"""Print every K0 probe (lanes per clock per SM) on the current GPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1110_2561_b200 import _native  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))  # noqa: E402
import knobs_env  # noqa: E402
knobs_env.apply()

NAMES = ["popc", "lop3", "iadd x2", "red spread", "red hashed 4033", "imad",
         "shf", "red 1 word", "red 2 lanes/word", "red 4 words 1 bank",
         "red 8 words x4 lanes", "red 1 word, vals 1|2^16",
         "red 2 lanes/word, vals 1|2^16"]
for i, n in enumerate(NAMES):
    lanes, mhz = _native.calibrate(i)
    print(f"{i:2d} {n:22s} {lanes:8.3f} lanes/clk/SM  ({mhz:.0f} MHz)")
