#!/bin/bash
cd "$(dirname "$0")/.."
for c in c3 c4; do for g in 3 4 5; do
  echo "== $c pair 3 gray $g"
  ISD_PAIR=3 ISD_GRAY=$g timeout 600 python tools/run_k1.py --config $c --reps 3 2>&1 | tail -2
done; done
