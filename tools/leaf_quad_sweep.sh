#!/bin/bash
# config 1 kernel variants (bench.py default line, kernel-only): one-warp-per-matrix band kernel vs the
# four-matrices-per-warp quad kernel (TRINV_LEAF32=quad) in several warps x slots shapes.  Alternating rounds.
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-fp64"
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(f\"{d['step_ms_stats']['median']:.4f} ms median  {d['value']:.4g} inv/s  frac {r['frac']:.4f}\")"; }
for round in 1 2; do  # QCFGS overrides the list
  echo -n "band           "; $B 2>/dev/null | show
  for q in ${QCFGS:-43 62 33 42 52 32 24}; do echo -n "quad qcfg=$q    "; TRINV_LEAF32=quad TRINV_LEAF32_QCFG=$q $B 2>/dev/null | show; done
done
