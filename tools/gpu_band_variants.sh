# banded plans forced on c3/c4 (ISD_BAND=1) and band spans on c5
for c in c3 c4; do echo "$c default"; python tools/run_k1.py --config $c --reps 4 2>&1 | grep "rep 3"
  echo "$c banded"; ISD_BAND=1 python tools/run_k1.py --config $c --reps 4 2>&1 | grep "rep 3"; done
for sp in 0 1 3; do echo "c5 span $sp"; ISD_BAND_SPAN=$sp python tools/run_k1.py --config c5 --reps 4 2>&1 | grep "rep 3"; done
