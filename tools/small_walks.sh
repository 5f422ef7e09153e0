#!/bin/bash
# small walks (c1, c2): device time of one full walk through the C ABI for
# forced pairing modes, loop widths and histogram copies per block
# (launch-, zero- and flush-bound)
cd "$(dirname "$0")/.."
for c in c2 c1; do
  echo "== $c default"; timeout 300 python tools/run_k1.py --config $c --reps 6 2>&1 | tail -3
  for p in 0 1 2; do for l in 0 2; do for h in 1 2 4 16; do
    echo "== $c pair $p loop $l nhist $h"
    ISD_PAIR=$p ISD_LOOP_BITS=$l ISD_NHIST_MAX=$h timeout 300 python tools/run_k1.py --config $c --reps 6 2>&1 | tail -2 | head -1
  done; done; done
done
