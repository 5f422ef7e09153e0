#!/bin/bash
cd "$(dirname "$0")/.."
for c in c4 c3 c5; do
  echo "== $c default"
  timeout 600 python tools/run_k1.py --config $c --reps 3 2>&1 | tail -2
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -n 2 2>&1 | tail -2
