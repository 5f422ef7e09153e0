# Gray width sweep (ISD_GRAY) on the BASELINE N=36 lattices, then the GPU
# fuzz of every Gray width x pairing mode against the C oracle
mkdir -p gpurun_out
for g in 2 3 4 5; do
  for c in c5 c3 c4; do
    echo "gray $g $c"
    ISD_GRAY=$g python tools/run_k1.py --config $c --reps 4 2>&1 | tail -2 | head -1
  done
  ISD_GRAY=$g python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 4 2>&1 | tail -2 | head -1
done 2>&1 | tee gpurun_out/k1_u.log
python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider -k "gray or band" \
  > gpurun_out/gpu_tests_u.log 2>&1; echo "tests exit=$?" >> gpurun_out/gpu_tests_u.log
tail -3 gpurun_out/gpu_tests_u.log
