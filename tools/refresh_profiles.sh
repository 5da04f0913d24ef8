#!/bin/bash
# Round-end evidence: every bench line (no profiler), sweeps, ncu launch lists and
# --set full captures of the dominant kernels.  Outputs under gpurun_out/; the
# summaries worth keeping are copied to profiles/ by hand.
set -o pipefail
export BENCH_ALLOW_SHORT=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/steps.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/steps.log
: > gpurun_out/bench_all.jsonl
for c in 1 0 2 3 4 5; do
  timeout 900 python bench.py --config $c >> gpurun_out/bench_all.jsonl 2> gpurun_out/bench_c$c.err || echo "{\"config\": $c, \"failed\": true}" >> gpurun_out/bench_all.jsonl
done
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python tools/sweep_n.py > gpurun_out/sweep_n.txt 2>&1
timeout 300 python tools/sweep_batched.py > gpurun_out/sweep_batched.txt 2>&1
# launch lists (cold-cache, serialised)
CMD1="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
CMD0="python bench.py --config 0 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-graph"
CMD3="python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD1 > gpurun_out/ncu_l1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c0.csv $CMD0 > gpurun_out/ncu_l0.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD3 > gpurun_out/ncu_l3.log 2>&1
# full captures of the dominant kernels
ncu --set full --clock-control none --import-source on -k regex:leaf32_tma -s 3 -c 1 -o gpurun_out/full_leaf32 $CMD1 > gpurun_out/ncu_f1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:blk_kernel -s 3 -c 1 -o gpurun_out/full_blk $CMD0 > gpurun_out/ncu_f0.log 2>&1
TRINV_PRODUCTS=dmma ncu --set full --clock-control none --import-source on -k regex:dmma_level -s 10 -c 2 -o gpurun_out/full_dmma_c2 python tools/prof_one.py L 8192 > gpurun_out/ncu_f2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:oz2_gemm -c 2 -o gpurun_out/full_oz2_c2 python tools/prof_one.py L 8192 > gpurun_out/ncu_f2oz.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:oz2_gemm -s 12 -c 2 -o gpurun_out/full_oz2_c3 python tools/prof_one.py U 32768 > gpurun_out/ncu_f3oz.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"oz2_split|oz2_recon|oz2_colmax" -s 6 -c 4 -o gpurun_out/full_oz2aux_c3 python tools/prof_one.py U 32768 > gpurun_out/ncu_f3aux.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf64_tma -c 1 -o gpurun_out/full_leaf64 python tools/sweep_batched.py 64 > gpurun_out/ncu_f64.log 2>&1
for f in full_leaf32 full_blk full_dmma_c2 full_oz2_c2 full_oz2_c3 full_oz2aux_c3 full_leaf64; do
  [ -f gpurun_out/$f.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/$f.txt 2>&1
done
ls -la gpurun_out >> gpurun_out/steps.log
python tools/kprof.py A 16384 > gpurun_out/kprof_A16384.txt 2>&1
python tools/kprof.py L 8192 > gpurun_out/kprof_L8192.txt 2>&1
python tools/kprof.py G 16384 > gpurun_out/kprof_G16384.txt 2>&1
python tools/kprof.py U 32768 > gpurun_out/kprof_U32768.txt 2>&1
TRINV_PRODUCTS=dmma python tools/kprof.py U 32768 > gpurun_out/kprof_U32768_dmma.txt 2>&1
for c in 2 3 4 5; do timeout 900 python bench.py --config $c --products dmma >> gpurun_out/bench_dmma.jsonl 2>/dev/null; done
timeout 1500 python tests/accuracy_report.py > gpurun_out/accuracy_report.txt 2>&1
