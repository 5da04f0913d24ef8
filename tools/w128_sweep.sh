#!/bin/bash
# 128x128 vs 64x64 level tiles: TRINV_LEVEL_W128 = waves of 128-tiles required (default 2)
for w in 2 4 8 16 32; do
  for n in 4096 8192 16384; do
    TRINV_LEVEL_W128=$w python tools/timeline.py L $n 2>/dev/null | head -1 | sed "s/^/w128=$w  /"
  done
  TRINV_LEVEL_W128=$w python tools/strassen_inversion.py 2>/dev/null | grep "config3 U n=32768                 2\|config4 inv_from_lu n=16384       1" | sed "s/^/w128=$w  /"
done
