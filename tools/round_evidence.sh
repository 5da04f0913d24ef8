#!/bin/bash
# Round-end evidence (run under gpurun): tests, smoke, every bench line, ncu launch list of
# the default bench command, ncu --set full of the headline kernel.  Outputs in gpurun_out/.
set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/steps.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/steps.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?" >> gpurun_out/steps.log
: > gpurun_out/bench_configs.jsonl
for c in 0 2 3 4 5; do
  timeout 900 python bench.py --config $c >> gpurun_out/bench_configs.jsonl 2> gpurun_out/bench_c$c.err || echo "{\"config\": $c, \"failed\": true}" >> gpurun_out/bench_configs.jsonl
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 20 --warmup 5"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_default.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/steps.log
CMD1="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-fp64"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:leaf32_tma -s 3 -c 1 -o gpurun_out/full_leaf32 $CMD1 > gpurun_out/ncu_full_leaf32.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/steps.log
cat gpurun_out/steps.log
timeout 900 python tests/accuracy_report.py > gpurun_out/accuracy.txt 2>&1; echo "accuracy rc=$?" >> gpurun_out/steps.log
: > gpurun_out/sweep_n.txt
for n in 512 1024 2048 4096 8192; do for op in L U; do python tools/timeline.py $op $n 2>/dev/null | head -1 >> gpurun_out/sweep_n.txt; done; done
python tools/timeline.py L 2048 2>/dev/null >> gpurun_out/sweep_n.txt
cat gpurun_out/steps.log
