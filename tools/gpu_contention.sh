#!/bin/bash
# autotune + calibration while other processes share the GPU: three
# concurrent first walks on a fresh plan cache, then one walk alone on the
# cache they left (it must not have kept a disturbed calibration)
cd "$(dirname "$0")/.."
for i in 1 2; do
  export XDG_CACHE_HOME=/tmp/contend$i; rm -rf $XDG_CACHE_HOME
  for j in 1 2 3; do python tools/run_k1.py --config c5 --reps 6 > /tmp/contend_$j.log 2>&1 & done
  wait
  echo "== round $i: alone on the shared cache"
  python tools/run_k1.py --config c5 --reps 4 2>&1 | tail -2 | head -1
done
export XDG_CACHE_HOME=/tmp/contend_clean; rm -rf $XDG_CACHE_HOME
echo "== fresh cache, alone"
python tools/run_k1.py --config c5 --reps 4 2>&1 | tail -2 | head -1
for c in c3 c4; do python tools/run_k1.py --config $c --reps 4 2>&1 | tail -2 | head -1; done
python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 4 2>&1 | tail -2 | head -1
