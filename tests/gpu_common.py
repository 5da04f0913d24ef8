"""Shared helpers for the -m gpu parity tests (inputs from synth/, expected values
from oracle/; the CUDA path is reached only through paper_2307_07611_b200)."""
import numpy as np

import oracle
import synth

REL_TOL = 1e-10      # BASELINE.json north_star: elementwise (floored, C7)
RES_TOL = 1e-13      # ||T X - I||_F / (||T||_F ||X||_F)


def sample_columns(n, cfg, count=64):
    """6 fixed boundary columns of the top split + seeded distinct others."""
    fixed = sorted({c for c in (0, 1, n // 2 - 1, n // 2, n - 2, n - 1) if 0 <= c < n})
    rest = [c for c in range(n) if c not in fixed]
    rng = np.random.default_rng(1000 + cfg)
    k = min(count - len(fixed), len(rest))
    extra = rng.choice(rest, size=k, replace=False) if k > 0 else []
    return np.array(sorted(set(fixed) | set(int(c) for c in extra)), dtype=np.int64)


def check_full(T, X, uplo, unit=False, rel=REL_TOL, res=RES_TOL):
    R = oracle.trinv(T, uplo, unit)
    e = oracle.floored_rel_err(X, R)
    Tu = T.copy()
    if unit:
        np.fill_diagonal(Tu, 1.0)
    Tu = np.tril(Tu) if uplo == "L" else np.triu(Tu)
    rr = oracle.residual_ratio(Tu, X)
    assert e <= rel, f"floored rel err {e:.3e}"
    assert rr <= res, f"residual {rr:.3e}"
    # structural zeros of the opposite triangle are exactly 0
    opp = np.triu(X, 1) if uplo == "L" else np.tril(X, -1)
    assert np.all(opp == 0.0)
    return e, rr
