#!/bin/bash
# knob sweep of k1_hoisted on the GPU box: prints ms per full walk
for cfg in c5 c3 c4; do
  for ls in 0 5 10 15; do
    for hb in 36864 73728 110592; do
      echo -n "$cfg lane_shift=$ls hist_bytes=$hb: "
      ISD_LANE_SHIFT=$ls ISD_HIST_BYTES=$hb python tools/run_k1.py --config $cfg --reps 3 | tail -1
    done
  done
done
