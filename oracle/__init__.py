"""CPU oracle for the FP64 triangular-inverse hot path (arXiv 2307.07611).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no
code with the CUDA path (paper_2307_07611_b200/); see oracle.c's header for
the passages each routine writes out and DESIGN.md for the readings used.

The C library is built by build() (gcc -O2 -ffp-contract=off -fopenmp); this
wrapper only marshals numpy arrays.
"""
import ctypes
import os
import subprocess

import numpy as np

from .metrics import (floored_rel_err, residual_ratio, column_residual_ratio,  # noqa: F401
                      factored_column_residual_ratio)
from .hopscotch import hopscotch_series, hopscotch_count  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)


def build(force=False):
    """Compile oracle.c into liboracle.so (plain gcc, no FMA contraction)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
                               "-o", _SO, src])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        for name in ("oracle_crit_upper", "oracle_crit_lower"):
            getattr(L, name).argtypes = [_i64, _dp, _i64, _dp, _i64, ctypes.c_int]
        for name in ("oracle_crit_lower_batched", "oracle_crit_upper_batched"):
            getattr(L, name).argtypes = [_i64, _i64, _dp, _i64, _i64, _dp, _i64, _i64, ctypes.c_int]
        for name in ("oracle_pathsum_upper", "oracle_pathsum_lower"):
            getattr(L, name).argtypes = [_i64, _dp, _i64, _dp, _i64, ctypes.c_int]
            getattr(L, name).restype = ctypes.c_int
        L.oracle_columns.argtypes = [ctypes.c_char, _i64, _dp, _i64, ctypes.c_int, _i64, _lp, _dp]
        L.oracle_skul.argtypes = [_i64, _dp, _dp, _dp, _dp, _dp]
        L.oracle_skul.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_lu_columns.argtypes = [_i64, _dp, _i64, ctypes.c_int, _dp, _i64, ctypes.c_int,
                                        _i64, _lp, _dp]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp)


def _c(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def crit_upper(R, unit=False):
    """Upper inverse by CRIT / CRIT* (Alg. 3 / Alg. 2)."""
    R = _c(R); n = R.shape[0]
    S = np.empty_like(R)
    lib().oracle_crit_upper(n, _p(R), n, _p(S), n, int(unit))
    return S


def crit_lower(L, unit=False):
    """Lower inverse via the transpose of CRIT, i.e. forward substitution."""
    L = _c(L); n = L.shape[0]
    X = np.empty_like(L)
    lib().oracle_crit_lower(n, _p(L), n, _p(X), n, int(unit))
    return X


def trinv(T, uplo, unit=False):
    return crit_lower(T, unit) if uplo == "L" else crit_upper(T, unit)


def crit_batched(A, uplo="L", unit=False):
    """Per-matrix CRIT over a [B, n, n] array."""
    A = _c(A); B, n, _ = A.shape
    X = np.empty_like(A)
    f = lib().oracle_crit_lower_batched if uplo == "L" else lib().oracle_crit_upper_batched
    f(n, B, _p(A), n, n * n, _p(X), n, n * n, int(unit))
    return X


def pathsum(T, uplo, unit=False):
    """Brute-force Theorem 1 with R = DT; n <= 24."""
    T = _c(T); n = T.shape[0]
    X = np.empty_like(T)
    f = lib().oracle_pathsum_lower if uplo == "L" else lib().oracle_pathsum_upper
    rc = f(n, _p(T), n, _p(X), n, int(unit))
    if rc != 0:
        raise ValueError("pathsum is exponential; n <= 24 only")
    return X


def columns(T, uplo, cols, unit=False, ld=None):
    """Columns `cols` of T^{-1} by substitution; returns [len(cols), n]."""
    T = np.asarray(T)
    assert T.dtype == np.float64 and T.flags.c_contiguous
    n = T.shape[0]
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty((len(cols), n), dtype=np.float64)
    lib().oracle_columns(uplo.encode(), n, _p(T), T.shape[1] if ld is None else ld, int(unit),
                         len(cols), cols.ctypes.data_as(_lp), _p(out))
    return out


def lu_columns(L, U, cols, unit_l=True, unit_u=False):
    """Columns `cols` of U^{-1} L^{-1} = (LU)^{-1} (SKUL)."""
    assert L.dtype == np.float64 and L.flags.c_contiguous and U.flags.c_contiguous
    n = L.shape[0]
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty((len(cols), n), dtype=np.float64)
    lib().oracle_lu_columns(n, _p(L), n, int(unit_l), _p(U), n, int(unit_u), len(cols),
                            cols.ctypes.data_as(_lp), _p(out))
    return out


def skul(A):
    """SKUL (Alg. 5): (L, U, S, K, info) with A = L U (U unit), S = U^{-1}, K = L^{-1}."""
    A = _c(A); n = A.shape[0]
    L, U, S, K = (np.empty_like(A) for _ in range(4))
    info = lib().oracle_skul(n, _p(A), _p(L), _p(U), _p(S), _p(K))
    return L, U, S, K, info


def inv_general(A):
    """A^{-1} = S K from SKUL; the product is a plain library matmul."""
    L, U, S, K, info = skul(A)
    if info:
        raise ZeroDivisionError(f"zero pivot at {info}")
    return S @ K


def set_threads(n):
    """OpenMP thread count of the oracle's loops (timing legs only; results are identical)."""
    lib().oracle_set_threads(int(n))


def max_threads():
    return int(lib().oracle_max_threads())
