#!/bin/bash
# 32x32-tile consumer-warp layouts (TRINV_T32CFG) for the mid-size levels, graph-replayed calls
for c in 0 1 2 3; do
  for n in 512 1024 2048; do
    TRINV_T32CFG=$c python tools/timeline.py L $n 2>/dev/null | head -1 | sed "s/^/t32cfg=$c  /"
  done
done
for c in 1 2; do TRINV_T32CFG=$c python -m pytest tests/test_gpu_trinv.py -q -x 2>&1 | tail -1 | sed "s/^/t32cfg=$c parity: /"; done
