"""NEXT row f2 (general inverse from A) and the DMMA engine as a GEMM: parity of
trinv_gemm / lu_crout / inv_general against numpy products and the CPU oracle
(SKUL, Alg. 5)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402
from gpu_common import REL_TOL, RES_TOL, sample_columns  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
RNG = np.random.default_rng(11)


def gpu(M):
    return torch.from_numpy(np.ascontiguousarray(M)).to(DEV)


def gpu_even(M):
    """Device copy whose leading dimension is even (the engine's TMA requirement)."""
    r, c = M.shape[-2:]
    t = torch.zeros(M.shape[:-1] + (c + (c % 2),), dtype=torch.float64, device=DEV)
    t[..., :c] = gpu(M)
    return t[..., :c]


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (5, 7, 3), (128, 128, 128), (200, 130, 330), (1000, 600, 1200),
                                   (2048, 2048, 512)])
def test_gemm_dense(M, N, K):
    A = RNG.standard_normal((M, K)); B = RNG.standard_normal((K, N)); C0 = RNG.standard_normal((M, N))
    C = gpu(C0)
    P.gemm(gpu_even(A), gpu_even(B), C=C, alpha=-0.5, beta=2.0)
    ref = -0.5 * (A @ B) + 2.0 * C0
    assert np.max(np.abs(C.cpu().numpy() - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref))) * K ** 0.5


@pytest.mark.parametrize("n,N", [(1, 3), (37, 50), (128, 256), (300, 129), (1024, 700)])
@pytest.mark.parametrize("which", ["AL", "AU", "BL", "BU"])
def test_gemm_triangular(n, N, which):
    T = RNG.standard_normal((n, n))
    T = np.tril(T) if which[1] == "L" else np.triu(T)
    if which[0] == "A":
        B = RNG.standard_normal((n, N))
        C = P.gemm(gpu_even(T), gpu_even(B), struct_a=which[1]).cpu().numpy()
        ref = T @ B
    else:
        A = RNG.standard_normal((N, n))
        C = P.gemm(gpu_even(A), gpu_even(T), struct_b=which[1]).cpu().numpy()
        ref = A @ T
    assert np.max(np.abs(C - ref)) <= 1e-12 * n ** 0.5 * max(1.0, np.max(np.abs(ref)))


def test_gemm_batched():
    b, M, N, K = 7, 96, 80, 64
    A = RNG.standard_normal((b, M, K)); B = RNG.standard_normal((b, K, N))
    C = P.gemm(gpu(A), gpu(B)).cpu().numpy()
    assert np.max(np.abs(C - A @ B)) <= 1e-12 * K


@pytest.mark.parametrize("n", [1, 3, 40, 64, 65, 100, 128, 129, 200, 513, 1000])
def test_lu_crout_vs_skul(n):
    Lg = synth.host(n, seed=n, tag="L", diag="pos")
    Ug = synth.host(n, seed=n, tag="U", uplo="U", diag="one")
    A = Lg @ Ug
    LU = P.lu_crout(gpu_even(A), check=True).cpu().numpy()
    L, U, S, K, info = oracle.skul(A)
    assert info == 0
    assert oracle.floored_rel_err(np.tril(LU), L) <= REL_TOL
    assert oracle.floored_rel_err(np.triu(LU, 1) + np.eye(n), U) <= REL_TOL


@pytest.mark.parametrize("n", [1, 2, 5, 64, 65, 127, 128, 129, 300, 1000, 1500])
def test_inv_general_full(n):
    Lg = synth.host(n, seed=2 * n, tag="L", diag="pos")
    Ug = synth.host(n, seed=2 * n, tag="U", uplo="U", diag="one")
    A = Lg @ Ug
    X = P.inv_general(gpu(A), check=True).cpu().numpy()
    R = oracle.inv_general(A)
    assert oracle.floored_rel_err(X, R) <= REL_TOL
    assert oracle.residual_ratio(A, X) <= RES_TOL


def test_inv_general_paper_5x5(golden):
    g = golden("paper_5x5_factors.txt")
    X = P.inv_general(gpu(g["A"])).cpu().numpy()
    assert np.max(np.abs(X - np.linalg.inv(g["A"]))) <= 1e-13
    assert np.max(np.abs(X - g["S_skul"] @ g["K_skul"])) <= 2e-4  # printed S K


def test_inv_general_zero_pivot_and_layout():
    A = np.array([[0.0, 1.0], [1.0, 0.0]])
    with pytest.raises(P.SingularMatrixError):
        P.inv_general(gpu(A), check=True)
    n = 333
    Lg = synth.host(n, seed=9, tag="L", diag="pos"); Ug = synth.host(n, seed=9, tag="U", uplo="U", diag="one")
    A = Lg @ Ug
    big = torch.zeros((n, n + 3), dtype=torch.float64, device=DEV)  # odd ld
    big[:, :n] = gpu(A)
    X = P.inv_general(big[:, :n]).cpu().numpy()
    assert oracle.floored_rel_err(X, oracle.inv_general(A)) <= REL_TOL


@pytest.mark.parametrize("n", [8192, 5000, 16384])
def test_inv_general_n8192_sampled(n):
    """BASELINE-scale general inverse (8192, and 16384 whose top LU node runs its six
    triangle-times-full products by the quadrant recursion with Strassen) and a ragged order
    (5000: uneven LU splits, ragged merges in the inverse factors): 64 columns against the SKUL
    oracle, A X - I gate."""
    Lg = torch.empty((n, n), dtype=torch.float64, device=DEV)
    Ug = torch.empty_like(Lg)
    synth.device_fill(Lg, n, seed=5, tag="L", diag="pos")
    synth.device_fill(Ug, n, seed=5, tag="U", uplo="U", diag="one")
    A = Lg @ Ug  # library DGEMM, input construction only
    X = P.inv_general(A, check=True)
    cols = sample_columns(n, 5)
    cidx = torch.from_numpy(cols).to(DEV)
    Xs = X[:, cidx]
    E = A @ Xs
    E[cidx, torch.arange(len(cols), device=DEV)] -= 1.0
    rho = (torch.linalg.norm(E) / (torch.linalg.norm(A) * torch.linalg.norm(Xs))).item()
    ref = oracle.lu_columns(Lg.cpu().numpy(), Ug.cpu().numpy(), cols, unit_l=False, unit_u=True)
    assert oracle.floored_rel_err(Xs.T.contiguous().cpu().numpy(), ref, axis_cols=0) <= REL_TOL
    assert rho <= RES_TOL


@pytest.mark.parametrize("n", [4, 64, 132, 1000])
def test_gemm_strassen(n):
    A = RNG.standard_normal((n, n)); B = RNG.standard_normal((n, n))
    C = P.gemm_strassen(gpu(A), gpu(B)).cpu().numpy()
    assert np.max(np.abs(C - A @ B)) <= 1e-12 * n
