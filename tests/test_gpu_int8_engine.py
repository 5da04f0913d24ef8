"""Product engines of the level products (trinv_set_product_engine / trinv_gemm_oz): FP64
DMMA (the default) and the opt-in FP64-emulated (Ozaki-II) engine on the INT8 tensor cores
(16 moduli + CRT): parity with the CPU oracle at the same gates, exactness of the integer
products on integer data, and NaN / Inf propagation."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402
from gpu_common import REL_TOL, RES_TOL, check_full, sample_columns  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(params=["int8crt"])
def int8_engine(request):
    P.set_product_engine(request.param, min_block=256)
    yield request.param
    P.set_product_engine()  # library default


@pytest.mark.parametrize("digits", [0])
def test_gemm_oz_integer_exact(digits):
    """Small integer operands are represented exactly (residues of exact scaled integers).
    The CRT scheme evaluates C' / M as a 96-bit fixed-point fraction and multiplies by M in
    FP64 (oz2.cu): a few roundings of 2^-53, exact zeros."""
    rng = np.random.default_rng(3)
    A = rng.integers(-100, 101, (256, 512)).astype(np.float64)
    B = rng.integers(-100, 101, (512, 512)).astype(np.float64)
    C = P.gemm_oz(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), digits=digits).cpu().numpy()
    if digits:
        assert np.array_equal(C, A @ B)
    else:
        assert np.all(np.abs(C - A @ B) <= 2.0**-50 * np.abs(A @ B))


@pytest.mark.parametrize("digits", [0])
@pytest.mark.parametrize("struct", ["N", "AL", "AU", "BL", "BU"])
def test_gemm_oz_vs_dmma(struct, digits):
    rng = np.random.default_rng(7)
    M = N = K = 1024
    A = rng.uniform(-1, 1, (M, K)); B = rng.uniform(-1, 1, (K, N))
    kw = {}
    if struct == "AL": A = np.tril(A); kw["struct_a"] = "L"
    if struct == "AU": A = np.triu(A); kw["struct_a"] = "U"
    if struct == "BL": B = np.tril(B); kw["struct_b"] = "L"
    if struct == "BU": B = np.triu(B); kw["struct_b"] = "U"
    Ad, Bd = torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV)
    R = (A.astype(np.longdouble) @ B.astype(np.longdouble)).astype(np.float64)
    C = P.gemm_oz(Ad, Bd, digits=digits, **kw).cpu().numpy()
    scale = np.abs(A).max(1, keepdims=True) * np.abs(B).max(0, keepdims=True) * K
    assert np.max(np.abs(C - R) / scale) <= 1e-16
    # alpha / beta
    C0 = torch.from_numpy(rng.uniform(-1, 1, (M, N))).to(DEV)
    C1 = P.gemm_oz(Ad, Bd, C=C0.clone(), alpha=-2.0, beta=0.5, digits=digits, **kw).cpu().numpy()
    assert np.max(np.abs(C1 - (-2.0 * R + 0.5 * C0.cpu().numpy()))) <= 1e-12


@pytest.mark.parametrize("K", [32768, 40960])
def test_gemm_oz_crt_long_k(K):
    """The CRT variant takes u8 x u8 residue products up to K = 32768 (255^2 K < 2^31) and
    u8 x s8 (symmetric B residues) above: both sides of the switch, at the same bound as
    test_gemm_oz_vs_dmma."""
    rng = np.random.default_rng(K)
    M, N = 128, 256
    A = rng.uniform(-1, 1, (M, K)); B = rng.uniform(-1, 1, (K, N))
    R = (A.astype(np.longdouble) @ B.astype(np.longdouble)).astype(np.float64)
    C = P.gemm_oz(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), digits=0).cpu().numpy()
    scale = np.abs(A).max(1, keepdims=True) * np.abs(B).max(0, keepdims=True) * K
    assert np.max(np.abs(C - R) / scale) <= 1e-16


@pytest.mark.parametrize("n", [512, 1024, 2048, 3072])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_trinv_int8_engine_parity(int8_engine, n, uplo):
    T = synth.host(n, seed=n, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    f = P.trinv_lower if uplo == "L" else P.trinv_upper
    X = f(torch.from_numpy(T).to(DEV)).cpu().numpy()
    check_full(T, X, uplo)


def test_config2_int8_engine(int8_engine):
    n = 8192
    T = torch.empty((n, n), dtype=torch.float64, device=DEV)
    synth.device_fill(T, n, diag="signed")
    X = P.trinv_lower(T)
    cols = sample_columns(n, 2)
    Th = T.cpu().numpy()
    Xs = X[:, torch.from_numpy(cols).to(DEV)].T.contiguous().cpu().numpy()
    R = oracle.columns(Th, "L", cols)
    assert oracle.floored_rel_err(Xs, R, axis_cols=0) <= REL_TOL
    assert oracle.column_residual_ratio(np.tril(Th), Xs, cols) <= RES_TOL


def test_inv_from_lu_int8_engine(int8_engine):
    n = 2048
    L = synth.host(n, tag="L", diag="one")
    U = synth.host(n, tag="U", uplo="U", diag="pos")
    X = P.inv_from_lu(torch.from_numpy(L).to(DEV), torch.from_numpy(U).to(DEV), unit_l=True).cpu().numpy()
    cols = np.arange(n)
    R = oracle.lu_columns(L, U, cols, unit_l=True)  # y = L^-1 e_j, x = U^-1 y
    assert oracle.floored_rel_err(X.T, R, axis_cols=0) <= REL_TOL
    assert oracle.residual_ratio(L @ U, X) <= RES_TOL


@pytest.mark.parametrize("engine", ["dmma", "int8crt"])
@pytest.mark.parametrize("n,uplo,cfg", [(16384, "L", 2), (32768, "U", 3)])
def test_large_engines(n, uplo, cfg, engine):
    """Config 3 size (and n = 16384) on both product engines (the INT8 engine at its
    default 2048 threshold, the smaller levels on DMMA; "dmma" for every level): 64 sampled
    columns at the BASELINE gates."""
    P.set_product_engine(engine, min_block=2048)
    try:
        T = torch.empty((n, n), dtype=torch.float64, device=DEV)
        synth.device_fill(T, n, uplo=uplo, diag="signed" if uplo == "L" else "pos")
        X = (P.trinv_lower if uplo == "L" else P.trinv_upper)(T)
        cols = sample_columns(n, cfg)
        Xs = X[:, torch.from_numpy(cols).to(DEV)].T.contiguous().cpu().numpy()
        del X
        Th = T.cpu().numpy()
        R = oracle.columns(Th, uplo, cols)
        assert oracle.floored_rel_err(Xs, R, axis_cols=0) <= REL_TOL
        Tt = np.tril(Th) if uplo == "L" else np.triu(Th)
        assert oracle.column_residual_ratio(Tt, Xs, cols) <= RES_TOL
    finally:
        P.set_product_engine()


def test_gemm_oz_nonfinite_propagates():
    """A NaN in row i of A makes row i of C NaN; an Inf in column j of B makes column j of
    C NaN (Inf x 0 terms): the split kernels flag the row / column and the reconstruction
    writes NaN there, as an FP64 product would carry NaN / Inf; other entries unchanged."""
    rng = np.random.default_rng(21)
    M, N, K = 256, 512, 512
    A = rng.uniform(-1, 1, (M, K)); B = rng.uniform(-1, 1, (K, N))
    C0 = P.gemm_oz(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), digits=0).cpu().numpy()
    A[7, 100] = np.nan
    B[200, 33] = np.inf
    C = P.gemm_oz(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), digits=0).cpu().numpy()
    bad = np.zeros((M, N), bool); bad[7, :] = True; bad[:, 33] = True
    assert np.all(np.isnan(C[bad]))
    assert np.array_equal(C[~bad], C0[~bad])


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_int8_engine_nonfinite_input_falls_back(int8_engine, uplo, bad):
    """NaN / Inf inside the referenced triangle: the scaling guard sees it and the call runs
    on DMMA (bit for bit the DMMA result, NaN where DMMA puts NaN)."""
    n = 1024
    T = synth.host(n, seed=5, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    i, j = (700, 300) if uplo == "L" else (300, 700)
    T[i, j] = bad
    f = P.trinv_lower if uplo == "L" else P.trinv_upper
    X8 = f(torch.from_numpy(T).to(DEV)).cpu().numpy()
    P.set_product_engine("dmma")
    Xd = f(torch.from_numpy(T).to(DEV)).cpu().numpy()
    assert np.isnan(Xd).any()
    assert np.array_equal(np.isnan(X8), np.isnan(Xd))
    assert np.array_equal(X8[~np.isnan(X8)], Xd[~np.isnan(Xd)])
