# shard-aware plans (the layout model sees a shard's fixed top bits)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "band or baseline or full or shard" \
  > gpurun_out/gpu_tests_top.log 2>&1; echo "tests exit=$?" >> gpurun_out/gpu_tests_top.log
tail -2 gpurun_out/gpu_tests_top.log
for t in 1 0; do
  echo "ISD_PLAN_TOP=$t"
  for i in 0 1 2 3 4 5 6 7; do ISD_PLAN_TOP=$t python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | grep -A1 "rep 3"; done
done 2>&1 | tee gpurun_out/k1_top.log
python tools/run_k1.py --config c5 --reps 4 2>&1 | grep "rep 3"
