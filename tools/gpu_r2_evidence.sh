#!/bin/bash
# r2 evidence pass: GPU suite (release + bounds-checked subset), smoke, the
# reference's own suite on the drop-in, the bench line, launch list, ncu of
# the c5 walk (roofline traffic), of an 8-way shard and of K2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r2e}
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/${T}_gpu.log 2>&1; echo "suite rc=$?" >> gpurun_out/${T}_gpu.log
ISD_LIBRARY=paper_1110_2561_b200/libisingdos_b200_dbg.so timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -q -m gpu -x > gpurun_out/${T}_gpu_dbg.log 2>&1; echo "dbg suite rc=$?" >> gpurun_out/${T}_gpu_dbg.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
PYTHONPATH=.:tests timeout 1800 python -m pytest reference_suite -q -p refsuite_plugin -p no:cacheprovider -rxX > gpurun_out/${T}_reference_suite.txt 2>&1; echo "reference suite rc=$?" >> gpurun_out/${T}_reference_suite.txt
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?" >> gpurun_out/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --extra-configs "" --no-shard-emulation --no-cold --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_jit -s 2 -c 1 -o gpurun_out/${T}_k1_c5 python tools/run_k1.py --config c5 --reps 3 > gpurun_out/${T}_ncu_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_jit -s 2 -c 1 -o gpurun_out/${T}_k1_shard3 python tools/run_k1.py --config c5 --shards 8 --index 3 --reps 3 > gpurun_out/${T}_ncu_k1s.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_ -c 1 -o gpurun_out/${T}_k2_c5 python tools/k2_time.py --config c5 --reps 2 > gpurun_out/${T}_ncu_k2.log 2>&1
for f in gpu gpu_dbg smoke; do tail -n 2 gpurun_out/${T}_$f.log; done; tail -n 2 gpurun_out/${T}_reference_suite.txt gpurun_out/${T}_bench.err
