#!/bin/bash
# DMMA tile choice (TRINV_GEMM_WAVES = tiles per SM required before a larger tile) vs n.
for w in 2 1 0.5 0.25; do
  for n in 1024 2048 4096 8192; do
    TRINV_GEMM_WAVES=$w python tools/timeline.py L $n 2>/dev/null | head -1 | sed "s/^/waves=$w  /"
  done
done
