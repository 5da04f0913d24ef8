#!/bin/bash
# config 1 kernel variants (bench.py default line, kernel-only): one-warp-per-matrix band kernel vs the
# two-matrices-per-warp pair kernel in several warps x pair-slots shapes.  Two rounds, alternating.
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-fp64"
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(f\"{d['step_ms_stats']['median']:.4f} ms median  {d['value']:.4g} inv/s  frac {r['frac']:.4f}\")"; }
for round in 1 2; do
  echo -n "band           "; $B 2>/dev/null | show
  for p in 82 182 143 43 62 52; do echo -n "pair pcfg=$p    "; TRINV_LEAF32=pair TRINV_LEAF32_PCFG=$p $B 2>/dev/null | show; done
done
