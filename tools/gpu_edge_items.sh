# small items of the extreme popcount classes as second items of blocks 0, 1
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "band or baseline or full or shard" \
  > gpurun_out/gpu_tests_edge2.log 2>&1; echo "tests exit=$?" >> gpurun_out/gpu_tests_edge2.log
tail -2 gpurun_out/gpu_tests_edge2.log
ISD_PROBE=1 ISD_AUTOTUNE=0 python tools/run_k1.py --config c5 --reps 2 > gpurun_out/probe12_full.log 2>&1
ISD_PROBE=1 ISD_AUTOTUNE=0 python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 2 > gpurun_out/probe12_shard.log 2>&1
for r in 1 2; do python tools/run_k1.py --config c5 --reps 4 2>&1 | grep "rep 3"; done
for i in 0 1 2 3 4 5 6 7; do python tools/run_k1.py --config c5 --shards 8 --index $i --reps 4 2>&1 | grep "rep 3"; done
