"""NEXT row f3: Strassen's recursion in the dense quadrant products of the top merge and of
U^-1 L^-1 (trinv_set_strassen; the paper's P_TF recursion, Eq. PTFmbk, with
Strassen for P_FF, P:20 / P:46 / P:523).  Parity with the CPU oracle at the BASELINE gates
for 1 and 2 levels, lower / upper / inv_from_lu, small orders with the threshold lowered
(so every code path of the decomposition runs) and config 3 / config 4 at full size."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402
from gpu_common import REL_TOL, RES_TOL, check_full, sample_columns  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture
def strassen(request):
    levels, min_h = request.param
    P.set_strassen(levels, min_h)
    yield levels
    P.set_strassen()  # library default


@pytest.mark.parametrize("strassen", [(1, 64), (2, 64)], indirect=True)
@pytest.mark.parametrize("n", [512, 1024])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_strassen_top_merge_parity(strassen, n, uplo):
    T = synth.host(n, seed=n + 3, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    f = P.trinv_lower if uplo == "L" else P.trinv_upper
    X = f(torch.from_numpy(T).to(DEV)).cpu().numpy()
    check_full(T, X, uplo)


@pytest.mark.parametrize("strassen", [(1, 64), (2, 64)], indirect=True)
def test_strassen_inv_from_lu_parity(strassen):
    n = 1024
    L = synth.host(n, tag="L", diag="one")
    U = synth.host(n, tag="U", uplo="U", diag="pos")
    X = P.inv_from_lu(torch.from_numpy(L).to(DEV), torch.from_numpy(U).to(DEV), unit_l=True).cpu().numpy()
    R = oracle.lu_columns(L, U, np.arange(n), unit_l=True)
    assert oracle.floored_rel_err(X.T, R, axis_cols=0) <= REL_TOL
    assert oracle.residual_ratio(L @ U, X) <= RES_TOL


@pytest.mark.parametrize("strassen", [(1, 64), (2, 64)], indirect=True)
@pytest.mark.parametrize("sgn", [1.0, -1.0])
def test_strassen_exact_closed_form(strassen, sgn):
    """Unit lower bidiagonal with subdiagonal -s, s = +-1: X_ij = s^(i-j) (the single path of
    Thm 1).  Every Strassen sum and product stays an integer of magnitude <= n^2, so the
    decomposed top merge reproduces the closed form bit for bit (lower and, transposed, upper)."""
    n = 1024
    L = np.eye(n) - sgn * np.eye(n, k=-1)
    i, j = np.indices((n, n))
    ref = np.where(i >= j, sgn ** (i - j).astype(np.float64), 0.0)
    X = P.trinv_lower(torch.from_numpy(L).to(DEV)).cpu().numpy()
    assert np.array_equal(X, ref)
    Xu = P.trinv_upper(torch.from_numpy(L.T.copy()).to(DEV)).cpu().numpy()
    assert np.array_equal(Xu, ref.T)


@pytest.mark.parametrize("strassen", [(1, 4096), (2, 4096)], indirect=True)
def test_strassen_config3(strassen):
    n = 32768
    T = torch.empty((n, n), dtype=torch.float64, device=DEV)
    synth.device_fill(T, n, uplo="U", diag="pos")
    X = P.trinv_upper(T)
    cols = sample_columns(n, 3)
    Xs = X[:, torch.from_numpy(cols).to(DEV)].T.contiguous().cpu().numpy()
    del X
    Th = T.cpu().numpy()
    R = oracle.columns(Th, "U", cols)
    assert oracle.floored_rel_err(Xs, R, axis_cols=0) <= REL_TOL
    assert oracle.column_residual_ratio(np.triu(Th), Xs, cols) <= RES_TOL


@pytest.mark.parametrize("strassen", [(1, 4096)], indirect=True)
def test_strassen_config4(strassen):
    n = 16384
    Ld = torch.empty((n, n), dtype=torch.float64, device=DEV)
    Ud = torch.empty((n, n), dtype=torch.float64, device=DEV)
    synth.device_fill(Ld, n, tag="L", diag="one")
    synth.device_fill(Ud, n, tag="U", uplo="U", diag="pos")
    X = P.inv_from_lu(Ld, Ud)
    cols = sample_columns(n, 4)
    Xs = X[:, torch.from_numpy(cols).to(DEV)].T.contiguous().cpu().numpy()
    del X
    L, U = Ld.cpu().numpy(), Ud.cpu().numpy()
    R = oracle.lu_columns(L, U, cols, unit_l=True)
    assert oracle.floored_rel_err(Xs, R, axis_cols=0) <= REL_TOL
    assert oracle.factored_column_residual_ratio(L, U, Xs, cols) <= RES_TOL


@pytest.mark.parametrize("strassen", [(2, 64)], indirect=True)
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_strassen_with_staged_layouts(strassen, uplo):
    """Odd leading dimensions make the call stage A and X through the workspace, after W and
    the Strassen scratch: the three regions must not overlap (round 2 fixed an overlap of the
    staging copies with the INT8 scratch).  NaN in the padding columns must not leak."""
    n, ld = 1024, 1027
    T = synth.host(n, seed=21, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    big = np.full((n, ld), np.nan)
    big[:, :n] = T
    Ad = torch.from_numpy(big).to(DEV)[:, :n]
    Xbig = torch.full((n, ld), float("nan"), dtype=torch.float64, device=DEV)
    Xd = Xbig[:, :n]
    f = P.trinv_lower if uplo == "L" else P.trinv_upper
    f(Ad, out=Xd)
    X = Xd.cpu().numpy()
    check_full(T, X, uplo)
    assert np.all(np.isnan(Xbig[:, n:].cpu().numpy()))  # padding untouched
