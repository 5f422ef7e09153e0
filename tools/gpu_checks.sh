#!/bin/bash
# Everything run on the GPU box before a round ends:
#   1. the GPU test suite with the release library
#   2. the same suite with the bounds-checked library (traps on any shared-
#      histogram address outside a warp's histogram; compute-sanitizer is
#      closed on this pool)
#   3. smoke + a short bench line
set -e
python -m pytest tests -m gpu -q -p no:cacheprovider
ISD_LIBRARY=$PWD/paper_1110_2561_b200/libisingdos_b200_dbg.so \
  python -m pytest tests -m gpu -q -p no:cacheprovider
python __graft_entry__.py smoke
python bench.py --steps 5 --warmup 3 --extra-configs ""
