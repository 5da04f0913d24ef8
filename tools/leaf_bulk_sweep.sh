#!/bin/bash
# config 1: row stores from registers (default) vs staged bulk stores (TRINV_LEAF_BULK=1/2/3), alternating
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-fp64"
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(f\"{d['step_ms_stats']['median']:.4f} ms median  {d['value']:.4g} inv/s  frac {r['frac']:.4f}\")"; }
for round in 1 2; do
  for v in 0 1 2 3; do echo -n "bulk=$v  "; TRINV_LEAF_BULK=$v $B 2>/dev/null | show; done
done
