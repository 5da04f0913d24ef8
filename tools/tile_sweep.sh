#!/bin/bash
# forced level tile (TRINV_LEVEL_TILE) vs the default heuristic, graph-replayed calls
for t in 0 64 128; do
  for n in 1024 2048 4096 8192; do
    TRINV_LEVEL_TILE=$t python tools/timeline.py L $n 2>/dev/null | head -1 | sed "s/^/tile=$t  /"
  done
done
TRINV_LEVEL_TILE=64 python tools/timeline.py L 2048 2>&1 | grep -v -i warn
