"""NEXT row f3: is one level of Strassen worth it
for the dense FP64 products on B200?  Times C = A B with the DMMA GEMM and with
one Strassen level over it, and measures the componentwise error of both on
sampled rows against an 80-bit long-double reference computed on the host.

    python tools/strassen_experiment.py > profiles/r01_strassen.txt
"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_07611_b200 as P  # noqa: E402


def timed(fn, reps):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    torch.manual_seed(0)
    print(f"{'n':>6s} {'dmma ms':>9s} {'strassen ms':>12s} {'speedup':>8s} {'err dmma':>10s} {'err strassen':>13s}")
    for n in (2048, 4096, 8192, 16384):
        A = (torch.rand((n, n), dtype=torch.float64, device="cuda") * 2 - 1)
        B = (torch.rand((n, n), dtype=torch.float64, device="cuda") * 2 - 1)
        C1 = torch.empty_like(A); C2 = torch.empty_like(A)
        reps = 10 if n <= 8192 else 3
        t1 = timed(lambda: P.gemm(A, B, C=C1), reps)
        t2 = timed(lambda: P.gemm_strassen(A, B, C=C2), reps)
        rows = np.random.default_rng(n).choice(n, 4, replace=False)
        Ah = A[rows].cpu().numpy().astype(np.longdouble)
        Bh = B.cpu().numpy().astype(np.longdouble)
        ref = Ah @ Bh
        den = np.abs(Ah) @ np.abs(Bh)
        e1 = float(np.max(np.abs(C1[rows].cpu().numpy() - ref) / den))
        e2 = float(np.max(np.abs(C2[rows].cpu().numpy() - ref) / den))
        print(f"{n:6d} {t1:9.3f} {t2:12.3f} {t1 / t2:8.3f} {e1:10.2e} {e2:13.2e}", flush=True)
        del A, B, C1, C2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
