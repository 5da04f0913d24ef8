"""inv_general accuracy at one order (64 sampled columns against the oracle) and its time:
    python tools/general_check.py 16384"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import accuracy_report as R  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
e, r = R.general_case(n)
print(f"inv_general n={n}: floored-rel {e:.3e} residual {r:.3e}")
A = torch.rand((n, n), dtype=torch.float64, device="cuda") + n * torch.eye(n, dtype=torch.float64, device="cuda")
X = torch.empty_like(A)
for i in range(4):
    torch.cuda.synchronize(); t = time.perf_counter(); P.inv_general(A, out=X); torch.cuda.synchronize()
    if i: print(f"  {1e3 * (time.perf_counter() - t):.1f} ms")
