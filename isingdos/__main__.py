"""`python -m isingdos` runs the engine's command line."""
import sys

from paper_1110_2561_b200.cli import main

sys.exit(main())
