#!/bin/bash
# split-K levels on / off (TRINV_SPLITK), graph-replayed calls (tools/timeline.py first line)
for sk in 1 0; do
  for op in L U; do
    for n in 1024 2048 4096 8192 16384; do
      TRINV_SPLITK=$sk python tools/timeline.py $op $n 2>/dev/null | head -1 | sed "s/^/splitk=$sk  /"
    done
  done
done
