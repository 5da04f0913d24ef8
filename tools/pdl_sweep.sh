#!/bin/bash
# PDL on / off (TRINV_PDL) and the GEMM 128-tile threshold (TRINV_GEMM_W128), graph-replayed calls
for pdl in 1 0; do
  for n in 1024 2048 4096 8192; do
    TRINV_PDL=$pdl python tools/timeline.py L $n 2>/dev/null | head -1 | sed "s/^/pdl=$pdl  /"
  done
done
for w in 2 8 32; do
  TRINV_GEMM_W128=$w python tools/strassen_inversion.py 2>/dev/null | grep "config3 U n=32768                 2\|config4 inv_from_lu n=16384       1\|config2 L n=8192                  0" | sed "s/^/gemm_w128=$w  /"
done
