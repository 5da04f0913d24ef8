#!/bin/bash
# Run every bench configuration once (no profiler) and collect the JSON lines.
out=${1:-gpurun_out/bench_all.jsonl}
: > $out
for c in 1 0 2 4 3; do
  timeout 600 python bench.py --config $c ${BENCH_ARGS:-} >> $out 2> gpurun_out/bench_c$c.err || echo "{\"config\": $c, \"failed\": true}" >> $out
done
cat $out
