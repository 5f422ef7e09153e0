#!/bin/bash
cd "$(dirname "$0")/.."
for c in c4 c3; do
  echo "== $c default"
  timeout 600 python tools/run_k1.py --config $c --reps 3 2>&1 | tail -2
  echo "== $c banded mode 3"
  ISD_PAIR=3 ISD_BAND=1 timeout 600 python tools/run_k1.py --config $c --reps 3 2>&1 | tail -2
done
