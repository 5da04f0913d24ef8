"""Pins for the CPU oracle (oracle/): each check ties it to something other
than itself — values the paper prints, closed forms, exact integer identities,
brute force on tiny inputs, library special cases.  CPU only."""
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth

RNG = np.random.default_rng(20230714)


# --- P-a: the paper's 4x4 worked example, exact --------------------
def test_paper_4x4_example_upper(golden):
    g = golden("paper_4x4_example.txt")
    T, S = g["T"], g["S"]
    for unit in (True, False):
        assert np.array_equal(oracle.crit_upper(T, unit=unit), S)
        assert np.array_equal(oracle.pathsum(T, "U", unit=unit), S)
        cols = oracle.columns(T, "U", np.arange(4), unit=unit)
        assert np.array_equal(cols.T, S)


def test_paper_4x4_example_lower_transpose(golden):
    g = golden("paper_4x4_example.txt")
    L, X = g["T"].T.copy(), g["S"].T.copy()  # P:71 transpose law
    for unit in (True, False):
        assert np.array_equal(oracle.crit_lower(L, unit=unit), X)
        assert np.array_equal(oracle.pathsum(L, "L", unit=unit), X)
        assert np.array_equal(oracle.columns(L, "L", np.arange(4), unit=unit).T, X)


def test_paper_4x4_S14_terms():
    # S_14 = -1*1 + 2*2 + 4*5 - 1*2*3*5 ... the four H(1,4) paths.
    assert -1 + 2 * 2 + 4 * 5 - 2 * 3 * 5 == -7


# --- P-b: Hopscotch series (Ex. 1, Prop. 1, Cor. 1) ---------------------------
def test_hopscotch_listing_H15(golden):
    rows = [tuple(int(x) for x in r) for r in golden("hopscotch_H_1_5.txt")["_"]]
    got = oracle.hopscotch_series(1, 5)
    assert sorted(got) == sorted(rows) and len(got) == 8
    # the paper lists the 8 sequences longest first
    assert [len(r) for r in rows] == [len(r) for r in got]


@pytest.mark.parametrize("b", range(2, 15))
def test_hopscotch_count(b):
    assert oracle.hopscotch_count(1, b) == 2 ** (b - 2)  # Prop. 1


def test_hopscotch_translation():
    for a in range(1, 8):
        for b in range(a + 1, 10):
            for xi in range(0, 6):  # Cor. 1
                lhs = set(oracle.hopscotch_series(a + xi, b + xi))
                rhs = {tuple(v + xi for v in s) for s in oracle.hopscotch_series(a, b)}
                assert lhs == rhs
    assert oracle.hopscotch_series(3, 3) == []  # H(a0,a0) = empty


def test_pathsum_term_count_matches_prop1():
    # Entry (i,j) of a unit upper matrix whose strict upper entries are all 1 and
    # with sign-alternating weights removed: T_ab = -1 makes every term +1 in Eq. 6
    # ((-1)^(l-1) * (-1)^(l-1) = 1), so S_ij = |H(i,j)| = 2^(j-i-1).
    n = 10
    T = np.triu(-np.ones((n, n)), 1) + np.eye(n)
    S = oracle.pathsum(T, "U", unit=True)
    for i in range(n):
        for j in range(i + 1, n):
            assert S[i, j] == 2 ** (j - i - 1)
    assert np.array_equal(oracle.crit_upper(T, unit=True), S)


# --- P-c: Cor. 2 integer closure: exact integer identities ----------
def _int_unit_lower(n, rng, lo=-1, hi=1, diag=None):
    L = np.tril(rng.integers(lo, hi + 1, size=(n, n)), -1).astype(np.float64)
    d = np.ones(n) if diag is None else diag
    return L + np.diag(d)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13, 21, 32, 40, 48])
def test_integer_closure_exact(n):
    for _ in range(4):
        d = RNG.choice([-1.0, 1.0], size=n)
        L = _int_unit_lower(n, RNG, diag=d)
        X = oracle.crit_lower(L)
        assert np.all(X == np.round(X))  # integers
        Li = [[int(v) for v in r] for r in L]
        Xi = [[int(v) for v in r] for r in X]
        for i in range(n):  # L X = I in exact Python integer arithmetic
            for j in range(n):
                s = sum(Li[i][k] * Xi[k][j] for k in range(n))
                assert s == (1 if i == j else 0)
        U = L.T.copy()
        assert np.array_equal(oracle.crit_upper(U), X.T)
        assert np.array_equal(oracle.columns(U, "U", np.arange(n)).T, X.T)


def test_integer_exact_vs_fractions_gauss_jordan():
    # Independent exact inverse by Gauss-Jordan in rationals (SPEC S:230 style oracle).
    n = 7
    U = np.triu(RNG.integers(-3, 4, size=(n, n)), 1).astype(np.float64) + np.eye(n)
    M = [[Fraction(int(U[i, j])) for j in range(n)] + [Fraction(int(i == j)) for j in range(n)]
         for i in range(n)]
    for c in range(n - 1, -1, -1):
        for r in range(c):
            f = M[r][c]
            M[r] = [a - f * b for a, b in zip(M[r], M[c])]
    inv = np.array([[float(M[i][n + j]) for j in range(n)] for i in range(n)])
    for f in (lambda T: oracle.crit_upper(T, unit=True), lambda T: oracle.pathsum(T, "U", True)):
        assert np.array_equal(f(U), inv)


# --- P-d / P-e: closed forms ---------------------------------------------------
@pytest.mark.parametrize("s", [0.5, -0.5, 1.0, -1.0, 2.0, -2.0])
@pytest.mark.parametrize("n", [1, 2, 7, 33, 64])
def test_unit_bidiagonal_closed_form(n, s):
    # L = I - s*subdiag: the only H-path i -> i-1 -> ... -> j gives X_ij = s^(i-j).
    L = np.eye(n) - s * np.eye(n, k=-1)
    X = oracle.crit_lower(L)
    i, j = np.indices((n, n))
    ref = np.where(i >= j, float(s) ** (i - j).astype(np.float64), 0.0)
    assert np.array_equal(X, ref)
    assert np.array_equal(oracle.crit_upper(L.T.copy()), ref.T)


@pytest.mark.parametrize("n", [1, 2, 9, 64, 100])
def test_all_ones_lower(n):
    L = np.tril(np.ones((n, n)))
    ref = np.eye(n) - np.eye(n, k=-1)
    assert np.array_equal(oracle.crit_lower(L), ref)
    assert np.array_equal(oracle.crit_upper(L.T.copy()), ref.T)


# --- P-f: special cases ----------------------------------------------------------
def test_identity_and_diagonal():
    n = 17
    assert np.array_equal(oracle.crit_lower(np.eye(n)), np.eye(n))
    d = 1.0 + RNG.random(n)
    d *= RNG.choice([-1, 1], size=n)
    X = oracle.crit_lower(np.diag(d))
    assert np.array_equal(X, np.diag(1.0 / d))  # correctly rounded reciprocals
    assert np.array_equal(oracle.crit_upper(np.diag(d)), np.diag(1.0 / d))
    assert np.array_equal(oracle.crit_upper(np.diag([2.0, 5.0])), np.diag([0.5, 0.2]))


def test_2x2_closed_forms():
    # SPEC S:209 example and [[a,0],[c,b]]^-1 = [[1/a,0],[-c/(ab),1/b]].
    assert np.array_equal(oracle.crit_upper(np.array([[2.0, 4.0], [0.0, 4.0]])),
                          np.array([[0.5, -0.5], [0.0, 0.25]]))
    for _ in range(20):
        a, b, c = RNG.uniform(0.5, 2, 3) * RNG.choice([-1, 1], 3)
        X = oracle.crit_lower(np.array([[a, 0.0], [c, b]]))
        ref = np.array([[1 / a, 0.0], [-c / (a * b), 1 / b]])
        assert np.allclose(X, ref, rtol=4e-16, atol=0)


def test_block_diagonal_decouples():
    n1, n2 = 11, 13
    A = synth.host(n1, seed=1); B = synth.host(n2, seed=2)
    L = np.zeros((n1 + n2, n1 + n2)); L[:n1, :n1] = A; L[n1:, n1:] = B
    X = oracle.crit_lower(L)
    assert np.array_equal(X[:n1, :n1], oracle.crit_lower(A))
    assert np.array_equal(X[n1:, n1:], oracle.crit_lower(B))
    assert np.all(X[n1:, :n1] == 0)


# --- P-g: power-of-two scaling invariant ----------------------------------------
@pytest.mark.parametrize("k", [3, -7])
def test_pow2_scaling(k):
    L = synth.host(50, seed=9)
    assert np.array_equal(oracle.crit_lower(L * 2.0 ** k), oracle.crit_lower(L) * 2.0 ** -k)


# --- P-h / P-i: residual invariant; brute force vs recurrences --------------------
@pytest.mark.parametrize("n", [8, 16, 64, 256, 512])
def test_residual_random(n):
    L = synth.host(n, seed=n)
    X = oracle.crit_lower(L)
    assert oracle.residual_ratio(L, X) <= 1e-15
    U = synth.host(n, seed=n + 1, uplo="U", diag="pos")
    assert oracle.residual_ratio(U, oracle.crit_upper(U)) <= 1e-15


@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 9, 12])
def test_pathsum_vs_crit_real(n):
    for seed in range(3):
        L = synth.host(n, seed=100 + seed)
        P = oracle.pathsum(L, "L")
        C = oracle.crit_lower(L)
        assert oracle.floored_rel_err(P, C) <= 1e-14
        U = synth.host(n, seed=200 + seed, uplo="U", diag="pos")
        assert oracle.floored_rel_err(oracle.pathsum(U, "U"), oracle.crit_upper(U)) <= 1e-14


@pytest.mark.parametrize("n", [1, 5, 12])
def test_pathsum_vs_crit_integer_exact(n):
    for _ in range(10):
        U = np.triu(RNG.integers(-4, 5, size=(n, n)), 1).astype(np.float64) + np.eye(n)
        assert np.array_equal(oracle.pathsum(U, "U", unit=True), oracle.crit_upper(U, unit=True))
        assert np.array_equal(oracle.pathsum(U, "U", unit=False), oracle.crit_upper(U, unit=True))


# --- library special case: solve_triangular(T, I) -------------------------------
@pytest.mark.parametrize("n", [3, 31, 200])
def test_vs_scipy_solve_triangular(n):
    L = synth.host(n, seed=7 * n)
    ref = scipy.linalg.solve_triangular(L, np.eye(n), lower=True)
    assert oracle.floored_rel_err(oracle.crit_lower(L), ref) <= 1e-12
    U = synth.host(n, seed=7 * n + 1, uplo="U", diag="pos")
    ref = scipy.linalg.solve_triangular(U, np.eye(n), lower=False)
    assert oracle.floored_rel_err(oracle.crit_upper(U), ref) <= 1e-12
    Lu = synth.host(n, seed=3, diag="one")
    ref = scipy.linalg.solve_triangular(Lu, np.eye(n), lower=True, unit_diagonal=True)
    assert oracle.floored_rel_err(oracle.crit_lower(Lu, unit=True), ref) <= 1e-12


def test_unit_flag_ignores_stored_diagonal():
    L = synth.host(20, seed=4)
    L1 = L.copy(); np.fill_diagonal(L1, 1.0)
    Lg = L.copy(); np.fill_diagonal(Lg, np.nan)
    assert np.array_equal(oracle.crit_lower(Lg, unit=True), oracle.crit_lower(L1))
    assert np.array_equal(oracle.columns(Lg, "L", [0, 5, 19], unit=True),
                          oracle.columns(L1, "L", [0, 5, 19]))


@pytest.mark.parametrize("stored", [7.0, np.nan])
def test_unit_flag_ignores_stored_diagonal_every_routine(stored):
    """CRIT* (Alg. 2) takes the diagonal as 1 whatever is stored there: the upper,
    batched (lower and upper), column and path-sum routines with unit=True give bit for bit the
    result of the same matrix with an explicit unit diagonal (round-2 mutation check: a CRIT* that
    read the stored diagonal, or a batched upper routine that dropped the flag, passed the pins)."""
    n = 12
    U = synth.host(n, seed=6, uplo="U", diag="pos")
    U1 = U.copy(); np.fill_diagonal(U1, 1.0)
    Ug = U.copy(); np.fill_diagonal(Ug, stored)
    assert np.array_equal(oracle.crit_upper(Ug, unit=True), oracle.crit_upper(U1))
    assert np.array_equal(oracle.columns(Ug, "U", [0, 4, 11], unit=True), oracle.columns(U1, "U", [0, 4, 11]))
    assert np.array_equal(oracle.pathsum(Ug, "U", unit=True), oracle.pathsum(U1, "U"))
    for uplo, A in (("L", synth.host(n, batch=3, seed=2)), ("U", synth.host(n, batch=3, uplo="U", diag="pos"))):
        A1 = A.copy(); Ag = A.copy()
        idx = np.arange(n)
        A1[:, idx, idx] = 1.0
        Ag[:, idx, idx] = stored
        assert np.array_equal(oracle.crit_batched(Ag, uplo, unit=True), oracle.crit_batched(A1, uplo))


# --- P-k: transpose law; columns == full ----------------------------------------
def test_transpose_law_and_columns():
    n = 90
    L = synth.host(n, seed=11)
    X = oracle.crit_lower(L)
    # column substitution is the same arithmetic as crit_lower: bitwise
    assert np.array_equal(oracle.columns(L, "L", np.arange(n)).T, X)
    # CRIT row recurrence (S U = I) vs back substitution (U x = e_j): same definition
    Xu = oracle.crit_upper(L.T.copy())
    assert oracle.floored_rel_err(Xu, X.T) <= 1e-13
    assert oracle.floored_rel_err(oracle.columns(L.T.copy(), "U", np.arange(n)).T, X.T) <= 1e-13


def test_batched_equals_single():
    A = synth.host(32, batch=6, b0=3)
    Xb = oracle.crit_batched(A)
    for b in range(6):
        assert np.array_equal(Xb[b], oracle.crit_lower(A[b]))


# --- P-j: the paper's printed 5x5 factors, 4 decimals ---------------
def test_paper_5x5_printed_factors(golden):
    g = golden("paper_5x5_factors.txt")
    tol = 2e-4
    assert np.max(np.abs(oracle.crit_upper(g["R_sqr"]) - g["S_sqr"])) <= tol
    assert np.max(np.abs(oracle.crit_upper(g["U_skul"], unit=True) - g["S_skul"])) <= tol
    assert np.max(np.abs(oracle.crit_lower(g["L_skul"]) - g["K_skul"])) <= tol
    # S K = A^-1: inv_from_lu columns on the printed factors (L non-unit, U unit)
    cols = oracle.lu_columns(g["L_skul"], g["U_skul"], np.arange(5), unit_l=False, unit_u=True)
    assert np.max(np.abs(cols.T - np.linalg.inv(g["A"]))) <= tol
    assert np.max(np.abs(cols.T - g["S_skul"] @ g["K_skul"])) <= tol


def test_lu_columns_vs_library():
    n = 120
    L = synth.host(n, seed=5, tag="L", diag="one")
    U = synth.host(n, seed=5, tag="U", uplo="U", diag="pos")
    A = L @ U
    cols = np.array([0, 1, 59, 60, 118, 119])
    got = oracle.lu_columns(L, U, cols, unit_l=True)
    ref = np.linalg.solve(A, np.eye(n)[:, cols]).T
    assert oracle.floored_rel_err(got, ref, axis_cols=0) <= 1e-10
    # and via the full triangular inverses U^-1 L^-1
    full = oracle.crit_upper(U) @ oracle.crit_lower(L, unit=True)
    assert oracle.floored_rel_err(got, full[:, cols].T, axis_cols=0) <= 1e-12


# --- metric code ---------------------------------------------------------------
def test_metrics():
    R = np.array([[1.0, 0.0], [1e-9, 2.0]])
    X = R.copy(); X[1, 0] += 1e-12
    # floor = 1e-6 * max|col 0| = 1e-6 -> rel = 1e-12/1e-6
    assert abs(oracle.floored_rel_err(X, R) - 1e-6) < 1e-9
    assert oracle.residual_ratio(np.eye(3), np.eye(3)) == 0.0
    T = np.array([[2.0, 0.0], [1.0, 4.0]])
    Xc = oracle.columns(T, "L", [1])
    assert oracle.column_residual_ratio(T, Xc, [1]) == 0.0


# Hand-computed non-zero values for the metric code (reading C7/C8; the residual is the
# definition L X = I of the bordering inverse, and S K = A^-1).
# Each case is chosen so that a dropped sqrt, a swapped product order (X T for T X), a
# mean instead of a max over a batch, a mis-indexed identity column or the wrong column
# axis gives a different number.
def test_residual_ratio_hand_values():
    # T = diag(2, 1), X = diag(0.5, 1.1): T X - I = diag(0, 0.1)
    T = np.diag([2.0, 1.0]); X = np.diag([0.5, 1.1])
    assert oracle.residual_ratio(T, X) == pytest.approx(0.1 / (np.sqrt(5.0) * np.sqrt(1.46)), rel=1e-12)
    # T = [[2,0],[1,1]], X = [[.5,0],[-.4,1]]: T X = [[1,0],[.1,1]] (X T would give .2)
    T = np.array([[2.0, 0.0], [1.0, 1.0]]); X = np.array([[0.5, 0.0], [-0.4, 1.0]])
    want = 0.1 / np.sqrt(6.0 * 1.41)
    assert oracle.residual_ratio(T, X) == pytest.approx(want, rel=1e-12)
    # batch: max over the batch, not the mean (the identity pair contributes 0)
    Tb = np.stack([np.eye(2), T]); Xb = np.stack([np.eye(2), X])
    assert oracle.residual_ratio(Tb, Xb) == pytest.approx(want, rel=1e-12)


def test_column_residual_ratio_hand_values():
    T = np.array([[2.0, 0.0], [1.0, 1.0]])  # inverse [[.5, 0], [-.5, 1]]
    # column 0 given as [.5, -.4]: T x - e_0 = [0, .1]; ||T||_F = sqrt 6, ||x|| = sqrt .41
    assert oracle.column_residual_ratio(T, np.array([[0.5, -0.4]]), [0]) == pytest.approx(
        0.1 / np.sqrt(6.0 * 0.41), rel=1e-12)
    # columns (1, 0) in that order: column 1 given as [0, 1.2] (T x - e_1 = [0, .2]),
    # column 0 exact; the identity must be subtracted at rows cols[c]
    Xc = np.array([[0.0, 1.2], [0.5, -0.5]])
    assert oracle.column_residual_ratio(T, Xc, [1, 0]) == pytest.approx(
        0.2 / np.sqrt(6.0 * (1.44 + 0.25 + 0.25)), rel=1e-12)


def test_factored_column_residual_ratio_hand_values():
    # L = [[1,0],[2,1]], U = [[2,1],[0,1]]: A = L U = [[2,1],[4,3]], A^-1 = [[1.5,-.5],[-2,1]].
    # Column 0 given as [1.5, -2.1]: U x = [.9, -2.1], L (U x) = [.9, -.3], minus e_0 =
    # [-.1, -.3]; ||L||_F = ||U||_F = sqrt 6, ||x|| = sqrt 6.66
    L = np.array([[1.0, 0.0], [2.0, 1.0]]); U = np.array([[2.0, 1.0], [0.0, 1.0]])
    got = oracle.factored_column_residual_ratio(L, U, np.array([[1.5, -2.1]]), [0])
    assert got == pytest.approx(np.sqrt(0.1) / (6.0 * np.sqrt(6.66)), rel=1e-12)
    # (U (L x) would give [2.9, .9]); the exact inverse columns give 0
    assert oracle.factored_column_residual_ratio(L, U, np.array([[1.5, -2.0], [-0.5, 1.0]]), [0, 1]) == 0.0


def test_floored_rel_err_hand_values():
    # axis_cols=0: each ROW of the arrays is one column of the inverse, floor from its own max
    R = np.array([[1e-9, 2.0], [4.0, 1e-3]])
    X = R + np.array([[1e-12, 0.0], [0.0, 1e-12]])
    # row 0: den = max(1e-9, 1e-6 * 2) = 2e-6 -> 5e-7; row 1: den = max(1e-3, 4e-6) = 1e-3
    # -> 1e-9.  Max 5e-7 (flooring along the other axis would give 2.5e-7)
    assert oracle.floored_rel_err(X, R, axis_cols=0) == pytest.approx(5e-7, rel=1e-9)
    # default axis: columns are X[:, j]; col 0 = (1e-9, 4) floor 4e-6, col 1 = (2, 1e-3) floor 2e-6
    assert oracle.floored_rel_err(X, R) == pytest.approx(max(1e-12 / 4e-6, 1e-12 / 1e-3), rel=1e-9)
    # an all-zero reference column divides by 1 (absolute error)
    assert oracle.floored_rel_err(np.array([[0.0, 0.0], [3e-3, 0.0]]), np.zeros((2, 2))) == pytest.approx(3e-3)
    assert oracle.floored_rel_err(np.zeros((0, 3)), np.zeros((0, 3))) == 0.0


# --- NEXT row f2: SKUL (Alg. 5) ------------------------------------------
def test_skul_paper_5x5_printed(golden):
    g = golden("paper_5x5_factors.txt")
    L, U, S, K, info = oracle.skul(g["A"])
    assert info == 0
    for got, ref in ((L, g["L_skul"]), (U, g["U_skul"]), (S, g["S_skul"]), (K, g["K_skul"])):
        assert np.max(np.abs(got - ref)) <= 1e-4  # 4 printed decimals
    assert np.max(np.abs(oracle.inv_general(g["A"]) - np.linalg.inv(g["A"]))) <= 1e-14


@pytest.mark.parametrize("n", [1, 2, 7, 40, 150])
def test_skul_identities(n):
    Lg = synth.host(n, seed=n, tag="L", diag="pos")
    Ug = synth.host(n, seed=n, tag="U", uplo="U", diag="one")
    A = Lg @ Ug
    L, U, S, K, info = oracle.skul(A)
    assert info == 0
    assert np.allclose(L @ U, A, rtol=0, atol=1e-14)                # A = L U
    assert oracle.floored_rel_err(L, Lg) <= 1e-12                   # unique Crout factors
    assert oracle.floored_rel_err(np.triu(U, 1), np.triu(Ug, 1)) <= 1e-11
    assert np.all(np.diag(U) == 1.0)
    assert oracle.floored_rel_err(S, oracle.crit_upper(U, unit=True)) <= 1e-13  # S = U^-1
    assert oracle.floored_rel_err(K, oracle.crit_lower(L)) <= 1e-13             # K = L^-1
    assert oracle.residual_ratio(A, S @ K) <= 1e-15


def test_skul_integer_exact():
    # unit-diagonal integer L and U: every intermediate is an integer (Cor. 2), exact
    rng = np.random.default_rng(3)
    n = 12
    L = np.tril(rng.integers(-2, 3, size=(n, n)), -1).astype(float) + np.eye(n)
    U = np.triu(rng.integers(-2, 3, size=(n, n)), 1).astype(float) + np.eye(n)
    A = L @ U
    L2, U2, S, K, info = oracle.skul(A)
    assert info == 0 and np.array_equal(L2, L) and np.array_equal(U2, U)
    X = S @ K
    assert np.array_equal(X, np.round(X))
    Ai = [[int(v) for v in r] for r in A]
    Xi = [[int(v) for v in r] for r in X]
    for i in range(n):
        for j in range(n):
            assert sum(Ai[i][k] * Xi[k][j] for k in range(n)) == (i == j)


def test_skul_zero_pivot():
    A = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert oracle.skul(A)[4] == 1
