#!/bin/bash
# ncu evidence for the batched kernel (config 1) and the DMMA product kernel (config 2).
set -o pipefail
CMD1="python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0"
CMD2="python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0"
export BENCH_ALLOW_SHORT=1
$CMD1 > gpurun_out/plain_c1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD1 > gpurun_out/ncu_l1.log 2>&1
$CMD1 > gpurun_out/plain_c1b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:leaf_tma -s 3 -c 1 -o gpurun_out/prof_leaf $CMD1 > gpurun_out/ncu_f1.log 2>&1
$CMD2 > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $CMD2 > gpurun_out/ncu_l2.log 2>&1
$CMD2 > gpurun_out/plain_c2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dmma_level -s 46 -c 2 -o gpurun_out/prof_dmma $CMD2 > gpurun_out/ncu_f2.log 2>&1
ls -la gpurun_out/
