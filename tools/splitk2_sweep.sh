#!/bin/bash
# split-K with the last-chunk fix-up (TRINV_SPLITK=2), 32x32 tiles, chunk sizes; parity check at n = 2048
python tools/timeline.py L 2048 2>/dev/null | head -1 | sed "s/^/default  /"
for kc in 128 256 512; do
  for n in 1024 2048 4096; do
    TRINV_SPLITK=2 TRINV_SPLITK_T=32 TRINV_SPLITK_KC=$kc python tools/timeline.py L $n 2>/dev/null | head -1 | sed "s/^/fixup t32 kc=$kc  /"
  done
done
for n in 1024 2048; do
  TRINV_SPLITK=2 TRINV_SPLITK_T=64 python tools/timeline.py L $n 2>/dev/null | head -1 | sed "s/^/fixup t64 auto  /"
done
TRINV_SPLITK=2 TRINV_SPLITK_T=32 TRINV_SPLITK_KC=256 python tools/timeline.py L 2048 2>&1 | grep -v -i warn
TRINV_SPLITK=2 TRINV_SPLITK_T=32 TRINV_SPLITK_KC=256 python -m pytest tests/test_gpu_trinv.py -q -x 2>&1 | tail -2
