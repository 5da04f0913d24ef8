"""Error metrics used by every parity check (reading C7/C8).

floored relative error: |X - R| / max(|R|, floor * max_i |R_ij| per column j);
residual ratio: ||T X - I||_F / (||T||_F ||X||_F); for inverses from factors (reading C21)
the factored residual ||L (U X_S) - I_S||_F / (||L||_F ||U||_F ||X_S||_F).  Plain numpy, fp64.
Test infrastructure only.
"""
import numpy as np

FLOOR = 1e-6


def floored_rel_err(X, R, axis_cols=-1, floor=FLOOR):
    """Max floored relative error. X, R: [..., n, m] with columns along the last axis
    (col_axis=-1 means columns are X[..., :, j]); for column-sample arrays pass
    arrays shaped [ncols, n] with axis_cols=0 meaning each row is one column."""
    X = np.asarray(X, dtype=np.float64); R = np.asarray(R, dtype=np.float64)
    if X.size == 0:
        return 0.0
    if axis_cols == 0:
        colmax = np.max(np.abs(R), axis=-1, keepdims=True)
    else:
        colmax = np.max(np.abs(R), axis=-2, keepdims=True)
    den = np.maximum(np.abs(R), floor * colmax)
    den = np.where(den == 0, 1.0, den)
    return float(np.max(np.abs(X - R) / den))


def residual_ratio(T, X):
    """||T X - I||_F / (||T||_F ||X||_F) for one square pair or a batch [B, n, n] (max over batch)."""
    T = np.asarray(T, dtype=np.float64); X = np.asarray(X, dtype=np.float64)
    n = T.shape[-1]
    E = T @ X - np.eye(n)
    num = np.sqrt(np.sum(E * E, axis=(-2, -1)))
    den = np.sqrt(np.sum(T * T, axis=(-2, -1))) * np.sqrt(np.sum(X * X, axis=(-2, -1)))
    return float(np.max(num / den))


def column_residual_ratio(T, Xcols, cols):
    """Residual restricted to sampled columns: ||T X_S - I_S||_F / (||T||_F ||X_S||_F).
    Xcols: [ncols, n] (row c = column cols[c] of X)."""
    T = np.asarray(T, dtype=np.float64)
    n = T.shape[0]
    Xs = np.asarray(Xcols, dtype=np.float64).T  # n x ncols
    E = T @ Xs
    E[np.asarray(cols), np.arange(len(cols))] -= 1.0
    return float(np.linalg.norm(E) / (np.linalg.norm(T) * np.linalg.norm(Xs)))


def factored_column_residual_ratio(L, U, Xcols, cols):
    """rho_LU of reading C21: ||L (U X_S) - I_S||_F / (||L||_F ||U||_F ||X_S||_F) for the
    sampled columns S of X = (L U)^-1, with the product applied factor by factor (no formed
    A).  L, U: the factors as full arrays (a unit diagonal stored explicitly);
    Xcols: [ncols, n] (row c = column cols[c] of X)."""
    L = np.asarray(L, dtype=np.float64); U = np.asarray(U, dtype=np.float64)
    Xs = np.asarray(Xcols, dtype=np.float64).T  # n x ncols
    E = L @ (U @ Xs)
    E[np.asarray(cols), np.arange(len(cols))] -= 1.0
    return float(np.linalg.norm(E) / (np.linalg.norm(L) * np.linalg.norm(U) * np.linalg.norm(Xs)))
