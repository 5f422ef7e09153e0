#!/bin/bash
# small walks (c1, c2): device time of one full walk through the C ABI for
# forced loop widths and pairing modes (launch-, zero- and flush-bound)
cd "$(dirname "$0")/.."
for c in c2 c1; do
  echo "== $c default"; timeout 300 python tools/run_k1.py --config $c --reps 6 2>&1 | tail -3
  for p in 0 1 2; do for l in 0 2 4 6; do
    echo "== $c pair $p loop $l"
    ISD_PAIR=$p ISD_LOOP_BITS=$l timeout 300 python tools/run_k1.py --config $c --reps 6 2>&1 | tail -2 | head -1
  done; done
done
