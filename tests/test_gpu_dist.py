"""NEXT row f1 on the GPU kernels: trinv_split with two ranks sharing cuda:0
(gloo collectives staged through host memory; the ranks' kernels never wait on
each other), checked against the CPU oracle."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, uplo, q, transport="nccl"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2307_07611_b200.dist import trinv_split, trinv_split_p2p
        T = torch.empty((n, n), dtype=torch.float64, device="cuda:0")
        synth.device_fill(T, n, seed=4, uplo=uplo, diag="signed" if uplo == "L" else "pos")
        X = trinv_split(T, uplo) if transport == "nccl" else trinv_split_p2p(T, uplo)
        torch.cuda.synchronize()
        if rank == 0:
            Th = T.cpu().numpy()
            R = oracle.trinv(Th, uplo)
            Xh = X.cpu().numpy()
            ok = oracle.floored_rel_err(Xh, R) <= 1e-10 and oracle.residual_ratio(Th, Xh) <= 1e-13
            opp = np.triu(Xh, 1) if uplo == "L" else np.tril(Xh, -1)
            q.put(bool(ok and np.all(opp == 0)))
        else:
            q.put(X is None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("world,n,uplo", [(2, 1024, "L"), (2, 1500, "U"), (3, 2048, "L"), (3, 1000, "U"),
                                          (4, 2048, "U")])
def test_split_two_ranks_one_gpu(world, n, uplo, transport):
    """transport "nccl": process-group broadcast + gather (gloo here); "p2p": the kernels
    read A^-1 / B^-1 from and store the X21 panels into rank 0's X through CUDA IPC
    (peer memory), with barriers only."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, uplo, q, transport)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = [q.get(timeout=5) for _ in range(world)]
    assert all(results), results
    assert all(p.exitcode == 0 for p in procs)


def test_split_single_process():
    import oracle
    import synth
    from paper_2307_07611_b200.dist import trinv_split
    n = 3000
    T = torch.from_numpy(synth.host(n, seed=8)).cuda()
    X = trinv_split(T, "L").cpu().numpy()
    assert oracle.floored_rel_err(X, oracle.crit_lower(T.cpu().numpy())) <= 1e-10


def _worker_large(rank, world, port, n, uplo, q, transport):
    """As _worker at a size whose panel products take the INT8 CRT engine; 64 sampled
    columns against the oracle."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from gpu_common import REL_TOL, RES_TOL, sample_columns
        import paper_2307_07611_b200 as P
        from paper_2307_07611_b200.dist import trinv_split, trinv_split_p2p
        P.set_product_engine("int8crt", min_block=2048)  # the 2048-wide panels of n = 16384 over 2 ranks
        T = torch.empty((n, n), dtype=torch.float64, device="cuda:0")
        synth.device_fill(T, n, seed=6, uplo=uplo, diag="signed" if uplo == "L" else "pos")
        X = trinv_split(T, uplo) if transport == "nccl" else trinv_split_p2p(T, uplo)
        torch.cuda.synchronize()
        if rank == 0:
            cols = sample_columns(n, 2)
            Xs = X[:, torch.from_numpy(cols).to("cuda:0")].T.contiguous().cpu().numpy()
            Th = T.cpu().numpy()
            R = oracle.columns(Th, uplo, cols)
            Tt = np.tril(Th) if uplo == "L" else np.triu(Th)
            ok = (oracle.floored_rel_err(Xs, R, axis_cols=0) <= REL_TOL and
                  oracle.column_residual_ratio(Tt, Xs, cols) <= RES_TOL)
            q.put(bool(ok))
        else:
            q.put(X is None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_split_int8_panels(uplo, transport):
    """n = 16384 over two ranks: the 2048-wide panel products run on the INT8 CRT engine
    (block threshold lowered to 2048 in the workers; the input passes the scaling guard)."""
    world, n = 2, 16384
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_large, args=(r, world, port, n, uplo, q, transport)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    results = [q.get(timeout=5) for _ in range(world)]
    assert all(results), results
    assert all(p.exitcode == 0 for p in procs)


def test_split_int8_panels_single_process():
    """One process (no process group), n = 16384: two 8192-wide panels on the INT8 engine
    at the default threshold."""
    import oracle
    import synth
    from gpu_common import REL_TOL, RES_TOL, sample_columns
    from paper_2307_07611_b200.dist import trinv_split
    n = 16384
    T = torch.empty((n, n), dtype=torch.float64, device="cuda:0")
    synth.device_fill(T, n, seed=8, diag="signed")
    X = trinv_split(T, "L")
    cols = sample_columns(n, 2)
    Xs = X[:, torch.from_numpy(cols).to("cuda:0")].T.contiguous().cpu().numpy()
    Th = T.cpu().numpy()
    assert oracle.floored_rel_err(Xs, oracle.columns(Th, "L", cols), axis_cols=0) <= REL_TOL
    assert oracle.column_residual_ratio(np.tril(Th), Xs, cols) <= RES_TOL
