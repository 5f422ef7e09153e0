#!/bin/bash
# ground truth: full-walk time for forced layouts (A,B,P,window shift)
for cfg in ${CFGS:-c5 c4 c3}; do
  case $cfg in
    c5) lays="55,1,0,0 58,1,0,15 58,1,0,6 59,1,0,6 70,1,0,12 70,1,0,6 69,1,0,15 1,38,0,0 1,51,0,3 1,45,0,9";;
    c4) lays="37,1,0,0 1,38,0,9 1,51,0,3 1,58,0,6 58,1,0,0 59,1,0,3 37,1,0,3 1,37,0,0";;
    c3) lays="61,1,0,0 89,1,0,15 88,1,0,15 70,1,0,12 1,69,0,15 83,1,0,15 71,1,0,0 1,76,0,0";;
  esac
  for l in $lays; do
    echo -n "$cfg $l: "; ISD_AUTOTUNE=0 ISD_COPY_VARIANT=low ISD_LAYOUT=$l python tools/run_k1.py --config $cfg --reps 3 | grep "rep 2"
  done
done
