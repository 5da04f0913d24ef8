"""The public calls under CUDA graph capture: the captured work (including inv_general's
forked second-stream branches and the INT8 engine's launches) replays to the same results
as eager calls, and replays see updated inputs in place."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402
from gpu_common import REL_TOL  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _capture(fn):
    fn(); torch.cuda.synchronize()  # first call outside capture (stream / tensor-map setup)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


@pytest.mark.parametrize("n", [64, 1000])
def test_trinv_graph_replay(n):
    T = torch.from_numpy(synth.host(n, seed=3, diag="signed")).to(DEV)
    X = torch.empty_like(T)
    g = _capture(lambda: P.trinv_lower(T, out=X))
    T.copy_(torch.from_numpy(synth.host(n, seed=4, diag="signed")).to(DEV))  # new input, same buffer
    g.replay(); torch.cuda.synchronize()
    ref = oracle.trinv(synth.host(n, seed=4, diag="signed"), "L")
    assert oracle.floored_rel_err(X.cpu().numpy(), ref) <= REL_TOL


def test_inv_general_graph_replay_with_forks():
    """n = 2048: the LU recursion forks its independent product pairs onto a second
    stream; the captured graph carries both branches."""
    n = 2048
    L = synth.host(n, seed=5, tag="L", diag="pos")
    U = synth.host(n, seed=5, tag="U", uplo="U", diag="one")
    A = torch.from_numpy(L @ U).to(DEV)
    X = torch.empty_like(A)
    eager = P.inv_general(A).cpu().numpy()
    g = _capture(lambda: P.inv_general(A, out=X))
    X.zero_()
    g.replay(); torch.cuda.synchronize()
    assert np.array_equal(X.cpu().numpy(), eager)  # same kernels, same order per element


def test_inv_from_lu_int8_graph_replay():
    n = 2048
    P.set_product_engine("int8crt", min_block=256)
    try:
        L = synth.host(n, tag="L", diag="one")
        U = synth.host(n, tag="U", uplo="U", diag="pos")
        Ld, Ud = torch.from_numpy(L).to(DEV), torch.from_numpy(U).to(DEV)
        X = torch.empty_like(Ld)
        g = _capture(lambda: P.inv_from_lu(Ld, Ud, unit_l=True, out=X))
        X.zero_()
        g.replay(); torch.cuda.synchronize()
        assert oracle.floored_rel_err(X.cpu().numpy(), np.linalg.inv(L @ U)) <= REL_TOL
    finally:
        P.set_product_engine()


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_strassen_paths_graph_replay(uplo):
    """The Strassen top merge and S K (forced down to n = 1024) under capture: the captured
    sequence of quadrant GEMMs, Strassen products and fused combinations replays to the
    eager result bit for bit, and on new input matches the oracle."""
    n = 1024
    P.set_strassen(2, 64)
    try:
        diag = "signed" if uplo == "L" else "pos"
        T = torch.from_numpy(synth.host(n, seed=3, uplo=uplo, diag=diag)).to(DEV)
        X = torch.empty_like(T)
        f = P.trinv_lower if uplo == "L" else P.trinv_upper
        eager = f(T).cpu().numpy()
        g = _capture(lambda: f(T, out=X))
        X.zero_()
        g.replay(); torch.cuda.synchronize()
        assert np.array_equal(X.cpu().numpy(), eager)
        T2 = synth.host(n, seed=4, uplo=uplo, diag=diag)
        T.copy_(torch.from_numpy(T2).to(DEV))
        g.replay(); torch.cuda.synchronize()
        assert oracle.floored_rel_err(X.cpu().numpy(), oracle.trinv(T2, uplo)) <= REL_TOL
        L = torch.from_numpy(synth.host(n, tag="L", diag="one")).to(DEV)
        U = torch.from_numpy(synth.host(n, tag="U", uplo="U", diag="pos")).to(DEV)
        Xg = torch.empty_like(L)
        eg = P.inv_from_lu(L, U, unit_l=True).cpu().numpy()
        gg = _capture(lambda: P.inv_from_lu(L, U, unit_l=True, out=Xg))
        Xg.zero_()
        gg.replay(); torch.cuda.synchronize()
        assert np.array_equal(Xg.cpu().numpy(), eg)
    finally:
        P.set_strassen()


def test_concurrent_calls_on_streams_and_threads():
    """Re-entrancy (include/trinv.h): calls from two host threads on two streams, each with
    its own buffers, overlap on the device and give the same bits as serial calls."""
    import threading
    n = 2048
    Ts = [torch.from_numpy(synth.host(n, seed=s, diag="signed")).to(DEV) for s in (11, 12)]
    ref = [P.trinv_lower(T).cpu().numpy() for T in Ts]
    Xs = [torch.empty_like(T) for T in Ts]
    streams = [torch.cuda.Stream() for _ in Ts]
    errs = []

    def work(i):
        try:
            with torch.cuda.stream(streams[i]):
                for _ in range(5):
                    P.trinv_lower(Ts[i], out=Xs[i], stream=streams[i])
            streams[i].synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for X, R in zip(Xs, ref):
        assert np.array_equal(X.cpu().numpy(), R)
