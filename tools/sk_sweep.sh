#!/bin/bash
# stream-K level launches (opt-in TRINV_SK=1) vs one CTA per tile (default): graph-replayed calls (tools/timeline.py)
t() { env $1 python tools/timeline.py L $2 2>/dev/null | head -1; }
for n in 1024 2048 4096 8192; do echo -n "sk=0  "; t TRINV_SK=0 $n; done
for tile in 64 6448 12864 128; do
  for bmin in 128 256 512; do
    for n in 1024 2048 4096 8192; do echo -n "tile=$tile bmin=$bmin  "; t "TRINV_SK=1 TRINV_SK_TILE=$tile TRINV_SK_BMIN=$bmin" $n; done
  done
done
for w in 4 16; do for n in 2048 4096; do echo -n "tile=12864 wmin=$w  "; t "TRINV_SK=1 TRINV_SK_TILE=12864 TRINV_SK_WMIN=$w TRINV_SK_BMIN=256" $n; done; done
TRINV_SK=1 TRINV_SK_TILE=12864 TRINV_SK_BMIN=256 python tools/timeline.py L 2048 2>/dev/null
