#!/bin/bash
# fused level launches (TRINV_FUSED) on / off, graph-replayed calls
for f in 1 0; do
  for op in L U; do
    for n in 512 1024 2048 4096 8192; do
      TRINV_FUSED=$f python tools/timeline.py $op $n 2>/dev/null | head -1 | sed "s/^/fused=$f  /"
    done
  done
done
python tools/timeline.py L 2048 2>&1 | grep -v -i warn
