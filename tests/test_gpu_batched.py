"""Parity of trinv_batched against the CPU oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402
from gpu_common import REL_TOL, RES_TOL  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _run(A, uplo="L", unit=False, **kw):
    X, info = P.trinv_batched(torch.from_numpy(A).to(DEV), uplo, unit=unit, info=True, **kw)
    torch.cuda.synchronize()
    return X.cpu().numpy(), info.cpu().numpy()


def test_config1_full_batch():
    """BASELINE config 1: 131072 lower 32x32, matrix b seeded by b; every matrix checked."""
    B = 131072
    A = synth.host(32, batch=B)
    X, info = _run(A)
    R = oracle.crit_batched(A)
    assert oracle.floored_rel_err(X, R) <= REL_TOL
    assert np.all(info == 0)
    idx = np.random.default_rng(0).choice(B, 512, replace=False)
    assert oracle.residual_ratio(A[idx], X[idx]) <= RES_TOL
    assert np.all(np.triu(X, 1) == 0.0)
    # device-generated input (the bench path) equals the host generator bitwise
    Ad = torch.empty((B, 32, 32), dtype=torch.float64, device=DEV)
    synth.device_fill(Ad, 32)
    assert torch.equal(Ad.cpu(), torch.from_numpy(A))


@pytest.mark.parametrize("n", [1, 2, 3, 7, 16, 17, 30, 31, 32, 33, 40, 47, 63, 64, 65, 80, 96, 113, 127, 128])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_orders_and_uplo(n, uplo):
    B = 8 * 148 * 2 + 5 if n <= 32 else 6 * 148 + 3  # several matrices per warp / CTA, ragged tail
    diag = "signed" if uplo == "L" else "pos"
    A = synth.host(n, batch=B, uplo=uplo, diag=diag)
    X, info = _run(A, uplo)
    assert oracle.floored_rel_err(X, oracle.crit_batched(A, uplo)) <= REL_TOL
    assert np.all(info == 0)
    opp = np.triu(X, 1) if uplo == "L" else np.tril(X, -1)
    assert np.all(opp == 0.0)


@pytest.mark.parametrize("uplo,n", [("L", 32), ("U", 32), ("U", 48), ("L", 64), ("L", 16), ("U", 13)])
def test_unit_ignores_diag_and_nan_other_triangle(uplo, n):
    B = 1000
    A = synth.host(n, batch=B, uplo=uplo)
    A1 = A.copy()
    idx = np.arange(n)
    A1[:, idx, idx] = 1.0
    poisoned = A.copy()
    poisoned[:, idx, idx] = np.nan
    tri = np.triu_indices(n, 1) if uplo == "L" else np.tril_indices(n, -1)
    poisoned[:, tri[0], tri[1]] = np.nan
    X, _ = _run(poisoned, uplo, unit=True)
    R = oracle.crit_batched(A1, uplo, unit=True)
    assert oracle.floored_rel_err(X, R) <= REL_TOL
    assert not np.isnan(X).any()


def test_exact_pins():
    # paper 4x4 inside a 32x32 identity-padded unit lower, bidiagonal s^(i-j), all-ones
    T = np.array([[1, 2, 4, 1], [0, 1, 3, 2], [0, 0, 1, 5], [0, 0, 0, 1]], dtype=np.float64)
    S = np.array([[1, -2, 2, -7], [0, 1, -3, 13], [0, 0, 1, -5], [0, 0, 0, 1]], dtype=np.float64)
    A = np.zeros((3, 32, 32))
    A[0] = np.eye(32); A[0, :4, :4] = T.T
    A[1] = np.eye(32) - 0.5 * np.eye(32, k=-1)
    A[2] = np.tril(np.ones((32, 32)))
    X, _ = _run(A)
    assert np.array_equal(X[0, :4, :4], S.T)
    i, j = np.indices((32, 32))
    assert np.array_equal(X[1], np.where(i >= j, 0.5 ** (i - j).astype(float), 0.0))
    assert np.array_equal(X[2], np.eye(32) - np.eye(32, k=-1))
    Xu, _ = _run(np.ascontiguousarray(np.transpose(A, (0, 2, 1))), "U")
    assert np.array_equal(Xu[0, :4, :4], S)
    # integer closure (Cor. 2): random unit +-1 lower, exact
    rng = np.random.default_rng(5)
    Ai = np.tril(rng.integers(-1, 2, size=(64, 32, 32)), -1).astype(np.float64) + np.eye(32)
    Xi, _ = _run(Ai)
    assert np.array_equal(Xi, oracle.crit_batched(Ai))
    # diagonal: correctly rounded reciprocals, bitwise
    d = 1.0 + rng.random((8, 32))
    Ad = np.zeros((8, 32, 32)); Ad[:, np.arange(32), np.arange(32)] = d
    Xd, _ = _run(Ad)
    assert np.array_equal(Xd[:, np.arange(32), np.arange(32)], 1.0 / d)


def test_strided_layouts_and_inplace():
    B, n, ld = 300, 32, 40
    A = synth.host(n, batch=B)
    big = np.full((B, n, ld), np.nan)
    big[:, :, :n] = A
    At = torch.from_numpy(big).to(DEV)[:, :, :n]  # ld = 40, stride = 1280
    X = P.trinv_batched(At)
    assert oracle.floored_rel_err(X.cpu().numpy(), oracle.crit_batched(A)) <= REL_TOL
    # odd leading dimension (plain-load path)
    big2 = np.zeros((B, n, 33)); big2[:, :, :n] = A
    X2 = P.trinv_batched(torch.from_numpy(big2).to(DEV)[:, :, :n])
    assert oracle.floored_rel_err(X2.cpu().numpy(), oracle.crit_batched(A)) <= REL_TOL
    # in place: X == A
    Ai = torch.from_numpy(A.copy()).to(DEV)
    P.trinv_batched(Ai, out=Ai)
    assert oracle.floored_rel_err(Ai.cpu().numpy(), oracle.crit_batched(A)) <= REL_TOL


def test_singular_info_and_determinism():
    B = 50
    A = synth.host(32, batch=B)
    A[7, 5, 5] = 0.0
    A[9, 31, 31] = 0.0
    A[9, 3, 3] = 0.0
    _, info = _run(A)
    assert info[7] == 6 and info[9] == 4 and info[0] == 0
    At = torch.from_numpy(synth.host(32, batch=4096)).to(DEV)
    X1 = P.trinv_batched(At); X2 = P.trinv_batched(At)
    assert torch.equal(X1, X2)
    # sub-batch gives the same bits (sharding invariance, P-l)
    X3 = P.trinv_batched(At[1000:1500].contiguous())
    assert torch.equal(X3, X1[1000:1500])


@pytest.mark.parametrize("uplo,n,B,chunk", [("L", 32, 20000, 0), ("U", 32, 9000, 1000), ("L", 17, 5000, 777),
                                            ("L", 48, 3000, 512), ("U", 100, 700, 128)])
def test_host_pipeline(uplo, n, B, chunk):
    """trinv_batched_host: host buffers, chunked H2D / invert / D2H pipeline (the e2e path)."""
    A = synth.host(n, batch=B, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    Ah = torch.from_numpy(A).pin_memory()
    X, info = P.trinv_batched_host(Ah, uplo, chunk=chunk, info=True)
    torch.cuda.synchronize()
    assert oracle.floored_rel_err(X.numpy(), oracle.crit_batched(A, uplo)) <= REL_TOL
    assert int(info.abs().sum()) == 0
    # the device path gives the same bits
    Xd = P.trinv_batched(torch.from_numpy(A).to(DEV), uplo)
    assert torch.equal(Xd.cpu(), X)
    # pageable memory works too (serialised copies), and in place X == A
    Ap = torch.from_numpy(A.copy())
    P.trinv_batched_host(Ap, uplo, out=Ap, chunk=chunk)
    torch.cuda.synchronize()
    assert torch.equal(Ap, X)


@pytest.mark.parametrize("n", [33, 64, 65, 100, 128])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_block_kernel_exact_pins_and_info(n, uplo):
    """Orders 33..128 (one CTA per matrix: 32-wide leaves + DMMA merges in shared memory):
    bidiagonal closed form s^(i-j) (P-d), diagonal reciprocals bitwise (C4), integer
    closure (Cor. 2, n <= 64), power-of-two scaling (P-g) and the zero-diagonal report."""
    i, j = np.indices((n, n))
    mats, want = [], []
    for s in (0.5, -0.5, 1.0, -1.0, 2.0):
        L = np.eye(n) - s * np.eye(n, k=-1)
        mats.append(L)
        want.append(np.where(i >= j, s ** (i - j).astype(float), 0.0))
    rng = np.random.default_rng(n)
    d = (1.0 + rng.random(n)) * rng.choice([-1.0, 1.0], n)
    mats.append(np.diag(d))
    want.append(np.diag(1.0 / d))
    A = np.stack(mats)
    if uplo == "U":
        A = np.ascontiguousarray(np.transpose(A, (0, 2, 1)))
        want = [w.T for w in want]
    X, info = _run(A, uplo)
    for b, w in enumerate(want):
        assert np.array_equal(X[b], w), b
    assert np.all(info == 0)
    if n <= 64:  # every intermediate an integer below 2^53: exact in any summation order
        Ai = np.tril(rng.integers(-1, 2, size=(16, n, n)), -1).astype(np.float64) + np.eye(n)
        if uplo == "U":
            Ai = np.ascontiguousarray(np.transpose(Ai, (0, 2, 1)))
        Xi, _ = _run(Ai, uplo)
        assert np.array_equal(Xi, oracle.crit_batched(Ai, uplo))
    G = synth.host(n, batch=40, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    X1, _ = _run(G, uplo)
    X8, _ = _run(G * 8.0, uplo)
    assert np.array_equal(X8 * 8.0, X1)
    G[3, n - 1, n - 1] = 0.0
    G[5, 7, 7] = 0.0
    G[5, n // 2, n // 2] = 0.0
    _, info = _run(G, uplo)
    assert info[3] == n and info[5] == 8 and info[0] == 0


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_batched64_tma_path(uplo):
    """n = 64 with a batch that fills the machine (>= 4096): the one-warp-per-matrix kernel
    with TMA-staged row bands (leaf64_tma_kernel); ragged count, zero-diagonal report,
    unit diagonal with a poisoned unreferenced triangle, and the same bits as the
    one-CTA-per-matrix path on a sub-batch below the threshold (P-l)."""
    n, B = 64, 5003
    A = synth.host(n, batch=B, uplo=uplo, diag="signed" if uplo == "L" else "pos")
    A[17, 40, 40] = 0.0
    A[4000, 3, 3] = 0.0
    A[4000, 60, 60] = 0.0
    X, info = _run(A, uplo)
    ok = np.ones(B, bool); ok[[17, 4000]] = False
    R = oracle.crit_batched(A[ok], uplo)
    assert oracle.floored_rel_err(X[ok], R) <= REL_TOL
    assert oracle.residual_ratio(A[ok][:256], X[ok][:256]) <= RES_TOL
    assert info[17] == 41 and info[4000] == 4 and np.count_nonzero(info) == 2
    opp = np.triu(X[ok], 1) if uplo == "L" else np.tril(X[ok], -1)
    assert np.all(opp == 0.0)
    # unit diagonal: neither the diagonal nor the other triangle is read
    Au = A.copy()
    idx = np.arange(n)
    Au[:, idx, idx] = np.nan
    tri = np.triu_indices(n, 1) if uplo == "L" else np.tril_indices(n, -1)
    Au[:, tri[0], tri[1]] = np.nan
    Xu, _ = _run(Au, uplo, unit=True)
    A1 = A.copy(); A1[:, idx, idx] = 1.0
    assert oracle.floored_rel_err(Xu[:300], oracle.crit_batched(A1[:300], uplo, unit=True)) <= REL_TOL
    assert not np.isnan(Xu).any()


_MMA_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle, synth, paper_2307_07611_b200 as P
from gpu_common import REL_TOL
bad = 0
for uplo in 'LU':
    A = synth.host(32, batch=4999, uplo=uplo, diag='signed' if uplo == 'L' else 'pos')  # odd: a lone last matrix
    X = P.trinv_batched(torch.from_numpy(A).cuda(), uplo).cpu().numpy()
    bad += oracle.floored_rel_err(X, oracle.crit_batched(A, uplo)) > REL_TOL
    opp = np.triu(X, 1) if uplo == 'L' else np.tril(X, -1)
    bad += not np.all(opp == 0.0)
    Ap = A.copy(); idx = np.arange(32); A1 = A.copy(); A1[:, idx, idx] = 1.0
    Ap[:, idx, idx] = np.nan
    tri = np.triu_indices(32, 1) if uplo == 'L' else np.tril_indices(32, -1)
    Ap[:, tri[0], tri[1]] = np.nan
    Xu = P.trinv_batched(torch.from_numpy(Ap).cuda(), uplo, unit=True).cpu().numpy()
    bad += oracle.floored_rel_err(Xu, oracle.crit_batched(A1, uplo, unit=True)) > REL_TOL
    Ai = torch.from_numpy(A.copy()).cuda(); P.trinv_batched(Ai, uplo, out=Ai)
    bad += not torch.equal(Ai.cpu(), torch.from_numpy(X))
A = synth.host(32, batch=64); A[5, 7, 7] = 0.0
_, info = P.trinv_batched(torch.from_numpy(A).cuda(), 'L', info=True)
bad += int(info[5].item()) != 8 or int(info[4].item()) != 0
print('BAD', bad)
"""


@pytest.mark.parametrize("mode,cfg", [("mma", "1063"), ("mma", "83"), ("pair", "82"), ("pair", "182"), ("pair", "43"),
                                      ("quad", "43"), ("quad", "62"), ("quad", "33")])
def test_leaf32_variant_parity(mode, cfg):
    """The opt-in n = 32 kernels (read once per process, hence a subprocess): the DMMA-merge
    kernel (TRINV_LEAF32=mma, pipelined and plain) and the two-matrices-per-warp kernel
    (TRINV_LEAF32=pair, half-row and full-row stores) against the oracle, lower / upper, an
    odd batch, unit diagonal with NaN-poisoned unreferenced entries, in place, zero-diagonal info."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TRINV_LEAF32=mode, TRINV_LEAF32_CFG=cfg, TRINV_LEAF32_PCFG=cfg, TRINV_LEAF32_QCFG=cfg)
    r = subprocess.run([sys.executable, "-c", _MMA_SCRIPT], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "BAD 0" in r.stdout, r.stdout + r.stderr[-2000:]
