"""`isingdos.cli` -> paper_1110_2561_b200.cli; `python -m isingdos.cli`
runs the engine's command line."""
import sys

from paper_1110_2561_b200 import cli as _impl

if __name__ == "__main__":
    sys.exit(_impl.main())
sys.modules[__name__] = _impl
