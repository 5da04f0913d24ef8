"""Out-of-bounds write guards (stand-in for compute-sanitizer, which is closed on this
pool): every output is placed inside a larger buffer filled with a sentinel, with
padding columns (ld > n), padding between batched matrices (stride > n*ld) and a
guard band after the last element; the call must leave every sentinel untouched and
still match the CPU oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402
from gpu_common import REL_TOL  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
SENT = -7.25e77  # exactly representable sentinel


def _guarded(rows, cols, ld, extra=64):
    """A (rows x cols) view with leading dimension ld inside a sentinel-filled buffer."""
    buf = torch.full((rows * ld + extra,), SENT, dtype=torch.float64, device=DEV)
    view = buf[: rows * ld].view(rows, ld)[:, :cols]
    return buf, view


def _inside_mask(rows, cols, ld, total):
    m = np.zeros(total, bool)
    for i in range(rows):
        m[i * ld: i * ld + cols] = True
    return m


def _assert_guards(buf, mask):
    b = buf.cpu().numpy()
    assert np.all(b[~mask] == SENT), f"{np.count_nonzero(b[~mask] != SENT)} guard values overwritten"


@pytest.mark.parametrize("n", [20, 33, 64, 100, 128, 129, 200, 1000])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_trinv_writes_stay_inside(n, uplo):
    T = synth.host(n, seed=n, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    ld = n + 6 if n % 2 == 0 else n + 3  # even and odd (staged) leading dimensions
    buf, X = _guarded(n, n, ld)
    f = P.trinv_lower if uplo == "L" else P.trinv_upper
    f(torch.from_numpy(T).to(DEV), out=X)
    torch.cuda.synchronize()
    assert oracle.floored_rel_err(X.cpu().numpy(), oracle.trinv(T, uplo)) <= REL_TOL
    _assert_guards(buf, _inside_mask(n, n, ld, buf.numel()))


@pytest.mark.parametrize("n,B", [(16, 700), (32, 700), (48, 300), (64, 300), (64, 4100), (100, 50)])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_batched_writes_stay_inside(n, B, uplo):
    A = synth.host(n, batch=B, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    ld = n + 2
    stride = n * ld + 4
    buf = torch.full((B * stride + 128,), SENT, dtype=torch.float64, device=DEV)
    X = torch.as_strided(buf, (B, n, n), (stride, ld, 1))
    P.trinv_batched(torch.from_numpy(A).to(DEV), uplo, out=X)
    torch.cuda.synchronize()
    assert oracle.floored_rel_err(X.cpu().numpy(), oracle.crit_batched(A, uplo)) <= REL_TOL
    mask = np.zeros(buf.numel(), bool)
    for b in range(B):
        for i in range(n):
            mask[b * stride + i * ld: b * stride + i * ld + n] = True
    _assert_guards(buf, mask)


@pytest.mark.parametrize("n", [100, 300])
def test_inv_from_lu_and_general_writes_stay_inside(n):
    L = synth.host(n, tag="L", diag="one")
    U = synth.host(n, tag="U", uplo="U", diag="pos")
    R = np.linalg.inv(L @ U)
    ld = n + 4
    buf, X = _guarded(n, n, ld)
    P.inv_from_lu(torch.from_numpy(L).to(DEV), torch.from_numpy(U).to(DEV), unit_l=True, out=X)
    torch.cuda.synchronize()
    assert oracle.floored_rel_err(X.cpu().numpy(), R) <= 1e-8
    _assert_guards(buf, _inside_mask(n, n, ld, buf.numel()))
    buf2, X2 = _guarded(n, n, ld)
    P.inv_general(torch.from_numpy(L @ U).to(DEV), out=X2)
    torch.cuda.synchronize()
    assert oracle.floored_rel_err(X2.cpu().numpy(), R) <= 1e-8
    _assert_guards(buf2, _inside_mask(n, n, ld, buf2.numel()))


@pytest.mark.parametrize("M,N,K", [(37, 50, 30), (130, 90, 70), (256, 300, 128)])  # even K, N: TMA operands
def test_gemm_writes_stay_inside(M, N, K):
    rng = np.random.default_rng(M)
    Ga, Gb = rng.random((M, K)), rng.random((K, N))
    ld = N + 2 + (N % 2)
    buf, C = _guarded(M, N, ld)
    P.gemm(torch.from_numpy(Ga).to(DEV), torch.from_numpy(Gb).to(DEV), C=C)
    torch.cuda.synchronize()
    assert np.max(np.abs(C.cpu().numpy() - Ga @ Gb)) <= 1e-12 * K
    _assert_guards(buf, _inside_mask(M, N, ld, buf.numel()))


@pytest.mark.parametrize("engine", ["int8crt"])
@pytest.mark.parametrize("n,uplo", [(1024, "L"), (1536, "U"), (2048, "L")])
def test_int8_engine_writes_stay_inside(engine, n, uplo):
    """The INT8 engine's kernels (residue splits into the workspace, the tensor-core GEMM,
    the reconstruction into X) inside the recursion, with the block threshold lowered so
    they carry the 512 / 1024 levels: X in a padded, guarded buffer."""
    P.set_product_engine(engine, min_block=256)
    try:
        T = synth.host(n, seed=n + 1, uplo=uplo, diag="signed" if uplo == "L" else "pos")
        ld = n + 8
        buf, X = _guarded(n, n, ld)
        f = P.trinv_lower if uplo == "L" else P.trinv_upper
        f(torch.from_numpy(T).to(DEV), out=X)
        torch.cuda.synchronize()
        assert oracle.floored_rel_err(X.cpu().numpy(), oracle.trinv(T, uplo)) <= REL_TOL
        _assert_guards(buf, _inside_mask(n, n, ld, buf.numel()))
    finally:
        P.set_product_engine()


@pytest.mark.parametrize("M,N,K,sa,sb", [(512, 768, 384, "N", "N"), (1024, 512, 1024, "L", "N"),
                                         (768, 1024, 1024, "N", "U")])
def test_gemm_oz_writes_stay_inside(M, N, K, sa, sb):
    rng = np.random.default_rng(M + N)
    Ga, Gb = rng.uniform(-1, 1, (M, K)), rng.uniform(-1, 1, (K, N))
    if sa == "L": Ga = np.tril(Ga)
    if sb == "U": Gb = np.triu(Gb)
    ld = N + 4
    buf, C = _guarded(M, N, ld)
    P.gemm_oz(torch.from_numpy(Ga).to(DEV), torch.from_numpy(Gb).to(DEV), C=C, struct_a=sa, struct_b=sb, digits=0)
    torch.cuda.synchronize()
    sc = np.abs(Ga).max(1, keepdims=True) * np.abs(Gb).max(0, keepdims=True) * K
    assert np.max(np.abs(C.cpu().numpy() - Ga @ Gb) / sc) <= 1e-15
    _assert_guards(buf, _inside_mask(M, N, ld, buf.numel()))
