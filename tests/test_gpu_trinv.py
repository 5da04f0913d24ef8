"""Parity of trinv_lower / trinv_upper / inv_from_lu
against the CPU oracle: full checks at sizes spanning several tiles and ragged
tails, sampled columns at BASELINE sizes, exact pins, layouts, errors."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402
from gpu_common import REL_TOL, RES_TOL, check_full, sample_columns  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def gpu(M):
    return torch.from_numpy(np.ascontiguousarray(M)).to(DEV)


def inv(T, uplo, **kw):
    f = P.trinv_lower if uplo == "L" else P.trinv_upper
    X = f(gpu(T), **kw)
    torch.cuda.synchronize()
    return X.cpu().numpy()


SIZES = [1, 2, 3, 31, 32, 33, 63, 64, 65, 96, 127, 128, 129, 200, 255, 256, 257, 384, 511, 640, 1000, 1024, 1500]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_full_parity(n, uplo):
    T = synth.host(n, seed=n, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    check_full(T, inv(T, uplo), uplo)


@pytest.mark.parametrize("n", [64, 300, 2048])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_unit_and_poisoned_other_triangle(n, uplo):
    T = synth.host(n, seed=3, uplo=uplo, diag="one")
    P_ = T.copy()
    np.fill_diagonal(P_, np.nan)
    mask = np.triu(np.ones((n, n), bool), 1) if uplo == "L" else np.tril(np.ones((n, n), bool), -1)
    P_[mask] = np.nan
    X = inv(P_, uplo, unit=True)
    check_full(T, X, uplo, unit=True)


def test_config0_n64():
    L = synth.host(64, seed=0)
    check_full(L, inv(L, "L"), "L")


def test_exact_pins_recursive():
    # bidiagonal closed form through every recursion level (P-d), integer closure (P-c)
    for n in (64, 257, 1024):
        for s in (0.5, -1.0, 2.0):
            nn = min(n, 60) if abs(s) == 2.0 else n
            L = np.eye(nn) - s * np.eye(nn, k=-1)
            i, j = np.indices((nn, nn))
            ref = np.where(i >= j, float(s) ** (i - j).astype(float), 0.0)
            assert np.array_equal(inv(L, "L"), ref)
            assert np.array_equal(inv(L.T, "U"), ref.T)
    rng = np.random.default_rng(7)
    for n in (33, 48):
        L = np.tril(rng.integers(-1, 2, size=(n, n)), -1).astype(np.float64) + np.diag(rng.choice([-1.0, 1.0], n))
        assert np.array_equal(inv(L, "L"), oracle.crit_lower(L))
        assert np.array_equal(inv(L.T, "U"), oracle.crit_upper(L.T.copy()))
    for n in (100, 700):
        assert np.array_equal(inv(np.tril(np.ones((n, n))), "L"), np.eye(n) - np.eye(n, k=-1))
        d = 1 + rng.random(n)
        assert np.array_equal(inv(np.diag(d), "L"), np.diag(1.0 / d))
    # block-diagonal (C = 0) -> X21 = 0 exactly
    A = synth.host(256, seed=1); B = synth.host(256, seed=2)
    L = np.zeros((512, 512)); L[:256, :256] = A; L[256:, 256:] = B
    X = inv(L, "L")
    assert np.all(X[256:, :256] == 0)


def test_pow2_scaling_and_transpose_law():
    L = synth.host(700, seed=21)
    X = inv(L, "L")
    assert np.array_equal(inv(L * 8.0, "L"), X / 8.0)
    Xu = inv(L.T, "U")
    assert oracle.floored_rel_err(Xu, X.T) <= REL_TOL


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_layouts_ld_and_misaligned(uplo):
    n = 333
    T = synth.host(n, seed=8, uplo=uplo, diag="pos")
    R = oracle.trinv(T, uplo)
    f = P.trinv_lower if uplo == "L" else P.trinv_upper
    for ld in (340, 333, 335):  # even ld > n, odd ld (staged)
        big = torch.full((n, ld), float("nan"), dtype=torch.float64, device=DEV)
        big[:, :n] = gpu(T)
        out = torch.full((n, ld + 2), float("nan"), dtype=torch.float64, device=DEV)
        X = f(big[:, :n], out=out[:, :n])
        assert oracle.floored_rel_err(X.cpu().numpy(), R) <= REL_TOL
    flat = torch.zeros(n * n + 1, dtype=torch.float64, device=DEV)  # 8-byte misaligned view
    Am = flat[1:].view(n, n)
    Am.copy_(gpu(T))
    assert oracle.floored_rel_err(f(Am).cpu().numpy(), R) <= REL_TOL


def test_singular_info_and_errors():
    L = synth.host(500, seed=2)
    L[321, 321] = 0.0
    L[400, 400] = 0.0
    with pytest.raises(P.SingularMatrixError) as e:
        P.trinv_lower(gpu(L), check=True)
    assert e.value.info == 322
    A = gpu(synth.host(100, seed=1))
    with pytest.raises(P.TrinvError):
        P.trinv_lower(A, out=A)  # aliasing


def test_determinism():
    A = gpu(synth.host(3000, seed=4))
    assert torch.equal(P.trinv_lower(A), P.trinv_lower(A))


@pytest.mark.parametrize("n,uplo", [(1000, "L"), (2048, "U"), (3000, "L")])
def test_graph_replay_matches_eager(n, uplo):
    """A call captured in a CUDA graph (its level launches become programmatic-dependency edges
    with PDL, the default) replays to the eager result bit for bit, and that result matches the
    oracle; replays on a dirtied output show nothing is read from a previous result."""
    A = synth.host(n, seed=9, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    Ad = gpu(A)
    f = P.trinv_lower if uplo == "L" else P.trinv_upper
    X_eager = f(Ad)
    Xg = torch.empty_like(Ad)
    f(Ad, out=Xg)  # warm-up outside capture (workspace sizing, kernel attributes)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f(Ad, out=Xg)
    for _ in range(3):
        Xg.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(Xg, X_eager)
    R = oracle.crit_lower(A) if uplo == "L" else oracle.crit_upper(A)
    assert oracle.floored_rel_err(Xg.cpu().numpy(), R) <= REL_TOL


def _sampled(T, X_dev, uplo, cfg, unit=False):
    n = T.shape[0]
    cols = sample_columns(n, cfg)
    Xs = X_dev[:, torch.from_numpy(cols).to(DEV)].T.contiguous().cpu().numpy()
    R = oracle.columns(T, uplo, cols, unit=unit)
    e = oracle.floored_rel_err(Xs, R, axis_cols=0)
    rr = oracle.column_residual_ratio(np.tril(T) if uplo == "L" else np.triu(T), Xs, cols)
    assert e <= REL_TOL, e
    assert rr <= RES_TOL, rr
    return e, rr


def test_config2_n8192_lower():
    n = 8192
    Ad = torch.empty((n, n), dtype=torch.float64, device=DEV)
    synth.device_fill(Ad, n)
    X = P.trinv_lower(Ad)
    T = Ad.cpu().numpy()
    assert np.array_equal(T[:64, :64], synth.host(n, seed=0)[:64, :64])
    _sampled(T, X, "L", 2)
    assert torch.all(torch.triu(X, 1) == 0)


@pytest.mark.parametrize("n,uplo", [(3000, "L"), (5000, "U"), (6144, "L"), (12345, "U")])
def test_sampled_ragged_large(n, uplo):
    """Orders that are not powers of two above the full-parity range: ragged last merges on the
    64x64 / 64x32 level tiles (and the 128-tile / quadrant decisions at their sizes), 64 oracle
    columns including the boundary columns of the top split."""
    Ad = torch.empty((n, n), dtype=torch.float64, device=DEV)
    synth.device_fill(Ad, n, uplo=uplo, diag="signed" if uplo == "L" else "pos", seed=n)
    X = (P.trinv_lower if uplo == "L" else P.trinv_upper)(Ad)
    T = Ad.cpu().numpy()
    assert np.array_equal(T[:48, :48], synth.host(n, seed=n, uplo=uplo, diag="signed" if uplo == "L" else "pos")[:48, :48])
    _sampled(T, X, uplo, 7)
    opp = torch.triu(X, 1) if uplo == "L" else torch.tril(X, -1)
    assert bool(torch.all(opp == 0))


@pytest.mark.slow
def test_config3_n32768_upper():
    n = 32768
    Ad = torch.empty((n, n), dtype=torch.float64, device=DEV)
    synth.device_fill(Ad, n, uplo="U", diag="pos")
    X = P.trinv_upper(Ad)
    torch.cuda.synchronize()
    T = Ad.cpu().numpy()
    del Ad
    _sampled(T, X, "U", 3)
    assert bool(torch.all(torch.tril(X[:4096, :4096], -1) == 0))


def test_inv_from_lu_ragged_sampled():
    """inv_from_lu at a ragged order (6000): 64 columns against the oracle's y = L^-1 e_j,
    x = U^-1 y, and the factored residual rho_LU (reading C21)."""
    n = 6000
    Ld = torch.empty((n, n), dtype=torch.float64, device=DEV)
    Ud = torch.empty((n, n), dtype=torch.float64, device=DEV)
    synth.device_fill(Ld, n, tag="L", diag="one")
    synth.device_fill(Ud, n, tag="U", uplo="U", diag="pos")
    X = P.inv_from_lu(Ld, Ud)
    cols = sample_columns(n, 8)
    Xs = X[:, torch.from_numpy(cols).to(DEV)].T.contiguous().cpu().numpy()
    L = Ld.cpu().numpy(); U = Ud.cpu().numpy()
    ref = oracle.lu_columns(L, U, cols, unit_l=True)
    assert oracle.floored_rel_err(Xs, ref, axis_cols=0) <= REL_TOL
    assert oracle.factored_column_residual_ratio(L, U, Xs, cols) <= RES_TOL


def test_inv_from_lu_small():
    for n in (64, 200, 1024):
        L = synth.host(n, seed=5, tag="L", diag="one")
        U = synth.host(n, seed=5, tag="U", uplo="U", diag="pos")
        X = P.inv_from_lu(gpu(L), gpu(U)).cpu().numpy()
        ref = oracle.lu_columns(L, U, np.arange(n), unit_l=True).T
        assert oracle.floored_rel_err(X, ref) <= REL_TOL
        A = L @ U
        assert oracle.residual_ratio(A, X) <= RES_TOL
    # paper's printed 5x5 SKUL factors: L non-unit, U unit
    from conftest import load_golden
    g = load_golden("paper_5x5_factors.txt")
    X = P.inv_from_lu(gpu(g["L_skul"]), gpu(g["U_skul"]), unit_l=False, unit_u=True).cpu().numpy()
    assert np.max(np.abs(X - np.linalg.inv(g["A"]))) <= 2e-4


def test_config4_inv_from_lu_n16384():
    n = 16384
    Ld = torch.empty((n, n), dtype=torch.float64, device=DEV)
    Ud = torch.empty((n, n), dtype=torch.float64, device=DEV)
    synth.device_fill(Ld, n, tag="L", diag="one")
    synth.device_fill(Ud, n, tag="U", uplo="U", diag="pos")
    X = P.inv_from_lu(Ld, Ud)
    Ad = Ld @ Ud  # library DGEMM, verification only (C21)
    cols = sample_columns(n, 4)
    cidx = torch.from_numpy(cols).to(DEV)
    Xs_dev = X[:, cidx]
    E = Ad @ Xs_dev
    E[cidx, torch.arange(len(cols), device=DEV)] -= 1.0
    rho_a = (torch.linalg.norm(E) / (torch.linalg.norm(Ad) * torch.linalg.norm(Xs_dev))).item()
    L = Ld.cpu().numpy(); U = Ud.cpu().numpy()
    del Ad, E
    Xs = Xs_dev.T.contiguous().cpu().numpy()
    ref = oracle.lu_columns(L, U, cols, unit_l=True)
    assert oracle.floored_rel_err(Xs, ref, axis_cols=0) <= REL_TOL
    assert rho_a <= RES_TOL, rho_a
    # rho_LU (reading C21): the factored residual L (U X_S) - I_S on the CPU, no formed A
    rho_lu = oracle.factored_column_residual_ratio(L, U, Xs, cols)
    assert rho_lu <= RES_TOL, rho_lu
