#!/bin/bash
# level tile shapes: forced 32x32 / 64x32 / 32x64 / 64x64 for every level, and the default rule
# (64x32 where 32x32 would run and >= TRINV_T6432_WAVES waves of 64x32 tiles; 0 = off)
for t in 6432 3264; do TRINV_LEVEL_TILE=$t timeout 300 python -m pytest tests/test_gpu_trinv.py -x -q 2>&1 | tail -1; done
timeout 300 python -m pytest tests/test_gpu_trinv.py -x -q 2>&1 | tail -1
for n in 1024 2048 4096 8192; do for op in L U; do
  for w in 0 2 3 4; do echo -n "w6432=$w "; TRINV_T6432_WAVES=$w python tools/timeline.py $op $n 2>/dev/null | head -1; done
done; done
python tools/timeline.py L 2048 2>/dev/null | tail -11
