"""Multi-process (gloo, world_size 2, CPU) checks of the batch partition and the
result gather used for BASELINE config 1 at N > 1 GPUs.  The per-shard inverse
here is the CPU oracle (test infrastructure), so the partition/gather logic of
paper_2307_07611_b200.dist is exercised without a GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_07611_b200.dist import gather_batched, shard_range


def test_shard_range_partitions_exactly():
    for B in (0, 1, 7, 131072, 131075):
        for W in (1, 2, 3, 4, 8):
            spans = [shard_range(B, W, r) for r in range(W)]
            assert spans[0][0] == 0
            for (a, c), (a2, _) in zip(spans, spans[1:]):
                assert a + c == a2
            assert sum(c for _, c in spans) == B
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        b0, cnt = shard_range(B, world, rank)
        A = synth.host(32, batch=cnt, b0=b0)  # generated locally from global indices
        X = torch.from_numpy(oracle.crit_batched(A))
        full = gather_batched(X, B)
        if rank == 0:
            ref = oracle.crit_batched(synth.host(32, batch=B))
            q.put(bool(np.array_equal(full.numpy(), ref)))
        else:
            q.put(full is None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [10, 33])
def test_gloo_world2_partition_and_gather(B):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = [q.get(timeout=5) for _ in range(world)]
    assert all(results), results
    assert all(p.exitcode == 0 for p in procs)


# --- NEXT row f1: one matrix split across ranks (partition + collectives, CPU stand-ins) ---
def _split_worker(rank, world, port, n, uplo, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2307_07611_b200.dist import trinv_split
        T = torch.from_numpy(synth.host(n, seed=3, uplo=uplo, diag="signed" if uplo == "L" else "pos"))

        def inv(M, u):
            return torch.from_numpy(oracle.trinv(M.contiguous().numpy(), u))

        def gemm(A, B, alpha, sa, sb):
            return alpha * (A @ B)

        X = trinv_split(T, uplo, inv=inv, gemm=gemm)
        if rank == 0:
            R = oracle.trinv(T.numpy(), uplo)
            q.put(oracle.floored_rel_err(X.numpy(), R) <= 1e-12 and oracle.residual_ratio(T.numpy(), X.numpy()) < 1e-15)
        else:
            q.put(X is None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,uplo", [(2, 300, "L"), (3, 257, "U"), (2, 128, "U"), (4, 520, "L"),
                                          (5, 700, "U")])
def test_gloo_split_single_matrix(world, n, uplo):
    """One matrix over `world` ranks: phase 1 recurses on halves of the group (sub-groups of
    1..3 ranks, the broadcast / gather sources translated to global ranks), phase 3 splits the
    off-diagonal block into 2G panels; rank 0 gets X equal to the oracle's."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, n, uplo, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    results = [q.get(timeout=5) for _ in range(world)]
    assert all(results), results
    assert all(p.exitcode == 0 for p in procs)
