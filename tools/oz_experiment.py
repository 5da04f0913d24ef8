"""INT8-tensor-core FP64 products (trinv_gemm_oz) vs the DMMA engine (trinv_gemm): error
against a long-double reference on small cases, error against DGEMM and time on large ones.

    python tools/oz_experiment.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_07611_b200 as P  # noqa: E402

DEV = "cuda:0"


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    rng = np.random.default_rng(0)
    # small: exact-ish reference in long double
    M, N, K = 256, 512, 384
    A = rng.uniform(-1, 1, (M, K)); B = rng.uniform(-1, 1, (K, N)) * np.exp(rng.normal(0, 3, (K, N)))
    R = (A.astype(np.longdouble) @ B.astype(np.longdouble)).astype(np.float64)
    Ad, Bd = torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV)
    scale = np.abs(A).max(1, keepdims=True) * np.abs(B).max(0, keepdims=True) * K
    for dg in (6, 7, 8, 9, 0):
        C = P.gemm_oz(Ad, Bd, digits=dg).cpu().numpy()
        print(f"small {M}x{N}x{K} {'crt' if dg == 0 else f'digits={dg}'}: max|err|/(K rowmax colmax) {np.max(np.abs(C - R) / scale):.2e}  "
              f"max rel {np.max(np.abs(C - R) / np.abs(R)):.2e}")
    C = P.gemm(Ad, Bd).cpu().numpy()
    print(f"small DMMA: max|err|/(K rowmax colmax) {np.max(np.abs(C - R) / scale):.2e}  max rel {np.max(np.abs(C - R) / np.abs(R)):.2e}")
    # large: time and error vs DGEMM (torch / cuBLAS)
    for n in (4096, 8192, 16384):
        A = torch.rand((n, n), dtype=torch.float64, device=DEV) * 2 - 1
        B = torch.rand((n, n), dtype=torch.float64, device=DEV) * 2 - 1
        R = A @ B
        t_d = timed(lambda: P.gemm(A, B), 3)
        for dg in (8, 0):
            C = P.gemm_oz(A, B, digits=dg)
            t = timed(lambda: P.gemm_oz(A, B, digits=dg), 3)
            err = (C - R).abs().max().item() / R.abs().max().item()
            print(f"dense n={n} {'crt16' if dg == 0 else f'digits={dg}'}: {t:8.2f} ms ({2 * n ** 3 / t / 1e9:7.1f} TF/s FP64-equiv)  "
                  f"DMMA {t_d:8.2f} ms ({2 * n ** 3 / t_d / 1e9:6.1f} TF/s)  max|C-R|/max|R| {err:.2e}")
        # triangular B (lower): k >= j blocks only
        Bl = torch.tril(B)
        Rl = A @ Bl
        t_dl = timed(lambda: P.gemm(A, Bl, struct_b="L"), 3)
        for dg in (8, 0):
            C = P.gemm_oz(A, Bl, struct_b="L", digits=dg)
            t = timed(lambda: P.gemm_oz(A, Bl, struct_b="L", digits=dg), 3)
            err = (C - Rl).abs().max().item() / Rl.abs().max().item()
            print(f"  tri-B n={n} {'crt16' if dg == 0 else f'digits={dg}'}: {t:8.2f} ms  DMMA {t_dl:8.2f} ms  "
                  f"speedup {t_dl / t:.2f}x  err {err:.2e}")
        del A, B, R, Bl, Rl, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
