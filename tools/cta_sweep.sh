#!/bin/bash
# full-walk time of the autotuned c5 plan vs shared-histogram budget per CTA
# (more histograms per CTA = fewer warps sharing one)
for hb in 36864 73728 110592; do
  for cap in 4 8 16; do
    echo -n "hist_bytes=$hb nhist_max=$cap: "
    ISD_HIST_BYTES=$hb ISD_NHIST_MAX=$cap python tools/run_k1.py --config c5 --reps 3 | grep "rep 2"
  done
done
