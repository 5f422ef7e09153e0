# banded c5 kernel: items per SM sweep and an ncu capture of the walk itself
# (ISD_AUTOTUNE=0: the model's best plan, which is the banded one, so the
# first k1_jit launch is the walk and not an autotune candidate)
mkdir -p gpurun_out
for ips in 2 3 4; do
  echo "items per SM: $ips"
  ISD_AUTOTUNE=0 ISD_BAND_ITEMS_PER_SM=$ips python tools/run_k1.py --config c5 --reps 4 2>&1 | tail -2
done 2>&1 | tee gpurun_out/k1_t.log
python tools/e2e_breakdown.py --config c5 --reps 10 2>&1 | tail -2 | tee -a gpurun_out/k1_t.log
ISD_AUTOTUNE=0 ncu --set full --clock-control none --import-source on -k regex:k1_jit -c 1 -f \
  -o gpurun_out/r1_k1_jit_band2_c5 python tools/run_k1.py --config c5 --reps 1 \
  > gpurun_out/ncu_t_c5.log 2>&1
tail -3 gpurun_out/ncu_t_c5.log
