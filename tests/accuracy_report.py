"""Floored relative error and residual of the product engines on the BASELINE configs 2-5
(64 sampled columns against the CPU oracle; test infrastructure, not part of pytest).

    python tests/accuracy_report.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402
from gpu_common import sample_columns  # noqa: E402

DEV = "cuda:0"


def tri_case(n, uplo, cfg):
    T = torch.empty((n, n), dtype=torch.float64, device=DEV)
    synth.device_fill(T, n, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    cols = sample_columns(n, cfg)
    X = (P.trinv_lower if uplo == "L" else P.trinv_upper)(T)
    Xs = X[:, torch.from_numpy(cols).to(DEV)].T.contiguous().cpu().numpy()
    del X
    Th = T.cpu().numpy()
    R = oracle.columns(Th, uplo, cols)
    Tt = np.tril(Th) if uplo == "L" else np.triu(Th)
    return oracle.floored_rel_err(Xs, R, axis_cols=0), oracle.column_residual_ratio(Tt, Xs, cols)


def lu_case(n):
    L = torch.empty((n, n), dtype=torch.float64, device=DEV)
    U = torch.empty_like(L)
    synth.device_fill(L, n, uplo="L", diag="one", tag="L")
    synth.device_fill(U, n, uplo="U", diag="pos", tag="U")
    X = P.inv_from_lu(L, U, unit_l=True)
    cols = sample_columns(n, 4)
    Xs = X[:, torch.from_numpy(cols).to(DEV)].T.contiguous().cpu().numpy()
    Lh, Uh = L.cpu().numpy(), U.cpu().numpy()
    R = oracle.lu_columns(Lh, Uh, cols, unit_l=True)
    # residual: rho_LU of reading C21, L (U X_S) - I_S applied factor by factor
    return oracle.floored_rel_err(Xs, R, axis_cols=0), oracle.factored_column_residual_ratio(Lh, Uh, Xs, cols)


def general_case(n):
    Lg = torch.empty((n, n), dtype=torch.float64, device=DEV)
    Ug = torch.empty_like(Lg)
    synth.device_fill(Lg, n, seed=5, tag="L", diag="pos")
    synth.device_fill(Ug, n, seed=5, tag="U", uplo="U", diag="one")
    A = Lg @ Ug  # library DGEMM, input construction only
    X = P.inv_general(A)
    cols = sample_columns(n, 5)
    cidx = torch.from_numpy(cols).to(DEV)
    Xs = X[:, cidx]
    E = A @ Xs
    E[cidx, torch.arange(len(cols), device=DEV)] -= 1.0
    rho = (torch.linalg.norm(E) / (torch.linalg.norm(A) * torch.linalg.norm(Xs))).item()
    R = oracle.lu_columns(Lg.cpu().numpy(), Ug.cpu().numpy(), cols, unit_l=False, unit_u=True)
    return oracle.floored_rel_err(Xs.T.contiguous().cpu().numpy(), R, axis_cols=0), rho


def main():
    for engine in ("dmma", "int8crt"):
        P.set_product_engine(engine, min_block=2048)
        for name, fn in (("config2 n=8192 L", lambda: tri_case(8192, "L", 2)),
                         ("config3 n=32768 U", lambda: tri_case(32768, "U", 3)),
                         ("config4 inv_from_lu n=16384", lambda: lu_case(16384)),
                         ("config5 inv_general n=16384", lambda: general_case(16384))):
            e, r = fn()
            print(f"{engine:8s} {name:28s} floored-rel {e:.3e}  residual {r:.3e}", flush=True)
    P.set_product_engine()


if __name__ == "__main__":
    main()
