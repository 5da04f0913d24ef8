"""Per-kernel breakdown of one INT8-engine product (tools/oz_prof.py n digits [struct_b])."""
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_07611_b200 as P  # noqa: E402

n, dg = int(sys.argv[1]), int(sys.argv[2])
sb = sys.argv[3] if len(sys.argv) > 3 else "N"
A = torch.rand((n, n), dtype=torch.float64, device="cuda") * 2 - 1
B = torch.rand((n, n), dtype=torch.float64, device="cuda") * 2 - 1
if sb == "L":
    B = torch.tril(B)
P.gemm_oz(A, B, digits=dg, struct_b=sb); torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    P.gemm_oz(A, B, digits=dg, struct_b=sb); torch.cuda.synchronize()
agg = defaultdict(float)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        agg[ev.name.split("(")[0][:50]] += ev.device_time_total / 1e3
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"  {v:9.3f} ms  {k}")
