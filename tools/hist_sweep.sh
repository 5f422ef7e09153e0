#!/bin/bash
# full-walk time vs shared histograms per CTA, at fixed layouts
export ISD_AUTOTUNE=0
for lay in 58,1,0,15 58,1,0,6 70,1,0,9; do
  for hb in 36864 73728 110592 147456; do
    echo -n "c5 layout=$lay hist_bytes=$hb: "
    ISD_LAYOUT=$lay ISD_HIST_BYTES=$hb python tools/run_k1.py --config c5 --reps 3 | grep "rep 2"
  done
done
