#!/bin/bash
# split-K on 32x32 tiles with fixed chunks (TRINV_SPLITK_T=32, TRINV_SPLITK_KC)
python tools/timeline.py L 2048 2>/dev/null | head -1 | sed "s/^/default  /"
for kc in 128 256 512; do
  for n in 1024 2048 4096; do
    TRINV_SPLITK=1 TRINV_SPLITK_T=32 TRINV_SPLITK_KC=$kc python tools/timeline.py L $n 2>/dev/null | head -1 | sed "s/^/t32 kc=$kc  /"
  done
done
TRINV_SPLITK=1 TRINV_SPLITK_T=32 TRINV_SPLITK_KC=256 python tools/timeline.py L 2048 2>&1 | grep -v -i warn
