#!/bin/bash
# level chain (default) vs one launch per product (TRINV_CHAIN=0): graph-replayed calls
for n in 512 1024 1500 2048 4096 8192; do for op in L U; do for c in 0 1; do
  echo -n "chain=$c "; TRINV_CHAIN=$c python tools/timeline.py $op $n 2>/dev/null | head -1
done; done; done
python tools/timeline.py L 2048 2>/dev/null
