"""NEXT row f3: Strassen levels in the dense quadrant products of the top merge / U^-1 L^-1,
measured inside whole inversions (time, floored relative error and residual against the
oracle on 64 sampled columns), DMMA engine.
    python tools/strassen_inversion.py > profiles/r02_strassen_inversion.txt"""
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402
from gpu_common import sample_columns  # noqa: E402

DEV = "cuda:0"


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def tri(n, uplo, cfg):
    T = torch.empty((n, n), dtype=torch.float64, device=DEV)
    synth.device_fill(T, n, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    X = torch.empty_like(T)
    f = P.trinv_lower if uplo == "L" else P.trinv_upper
    ms = timed(lambda: f(T, out=X))
    cols = sample_columns(n, cfg)
    Xs = X[:, torch.from_numpy(cols).to(DEV)].T.contiguous().cpu().numpy()
    Th = T.cpu().numpy()
    R = oracle.columns(Th, uplo, cols)
    Tt = np.tril(Th) if uplo == "L" else np.triu(Th)
    return ms, n ** 3 / 3, oracle.floored_rel_err(Xs, R, axis_cols=0), oracle.column_residual_ratio(Tt, Xs, cols)


def lu(n):
    L = torch.empty((n, n), dtype=torch.float64, device=DEV)
    U = torch.empty_like(L)
    synth.device_fill(L, n, tag="L", diag="one")
    synth.device_fill(U, n, tag="U", uplo="U", diag="pos")
    X = torch.empty_like(L)
    ms = timed(lambda: P.inv_from_lu(L, U, unit_l=True, out=X))
    cols = sample_columns(n, 4)
    Xs = X[:, torch.from_numpy(cols).to(DEV)].T.contiguous().cpu().numpy()
    Lh, Uh = L.cpu().numpy(), U.cpu().numpy()
    R = oracle.lu_columns(Lh, Uh, cols, unit_l=True)
    return ms, 4 * n ** 3 / 3, oracle.floored_rel_err(Xs, R, axis_cols=0), \
        oracle.factored_column_residual_ratio(Lh, Uh, Xs, cols)


def main():
    print("# Strassen levels in the dense quadrant products (DMMA engine), one B200; ms = median of 3")
    print(f"{'case':28s} {'levels':>6s} {'min_h':>6s} {'ms':>9s} {'TF/s':>7s} {'floored-rel':>12s} {'residual':>10s}")
    cases = [("config2 L n=8192", lambda: tri(8192, "L", 2), 2048),
             ("config3 U n=32768", lambda: tri(32768, "U", 3), 4096),
             ("config4 inv_from_lu n=16384", lambda: lu(16384), 4096)]
    for name, fn, mh in cases:
        for levels in (0, 1, 2):
            P.set_strassen(levels, mh)
            ms, fl, e, r = fn()
            print(f"{name:28s} {levels:6d} {mh:6d} {ms:9.3f} {fl / ms / 1e9:7.2f} {e:12.3e} {r:10.3e}", flush=True)
            torch.cuda.empty_cache()
    P.set_strassen()


if __name__ == "__main__":
    main()
