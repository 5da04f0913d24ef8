"""Multi-GPU partition of batched inverses (BASELINE config 1).

One process per GPU (torchrun).  Independent matrices are partitioned by batch:
rank r owns the contiguous global index range shard_range(B, world, r); its
shard is inverted locally by trinv_batched with no communication on the data
path (matrices are independent: P:160).  A collective is used only
to bring results to one rank when the caller asks for them (gather_batched),
and that transfer is timed apart from the throughput (bench.py).

Single large matrices are not split across GPUs ("replicas only"): each GPU
inverts its own matrix.
"""
import torch
import torch.distributed as dist


def shard_range(batch, world, rank):
    """Contiguous [b0, b0 + count) of `batch` matrices for `rank` (balanced to within one)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(batch, world)
    b0 = rank * base + min(rank, extra)
    return b0, base + (1 if rank < extra else 0)


def batched(A_local, uplo="L", unit=False, out=None, stream=None):
    """Invert this rank's shard [count, n, n] on its GPU (no communication)."""
    from . import trinv_batched
    return trinv_batched(A_local, uplo, unit=unit, out=out, stream=stream)


def gather_batched(X_local, batch, group=None, dst=0):
    """Collect every rank's shard into a [batch, n, n] tensor on rank `dst` (None elsewhere).

    Uses one all_gather_into_tensor over equal-size padded shards (NCCL on GPU
    tensors, gloo on CPU tensors), then drops the padding on `dst`.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = X_local.shape[-1]
    counts = [shard_range(batch, world, r)[1] for r in range(world)]
    cmax = max(counts)
    send = X_local
    if X_local.shape[0] != cmax:
        send = torch.zeros((cmax, n, n), dtype=X_local.dtype, device=X_local.device)
        send[: X_local.shape[0]] = X_local
    recv = torch.empty((world * cmax, n, n), dtype=X_local.dtype, device=X_local.device)
    dist.all_gather_into_tensor(recv, send.contiguous(), group=group)
    if rank != dst:
        return None
    parts = [recv[r * cmax: r * cmax + counts[r]] for r in range(world)]
    return torch.cat(parts, dim=0)


# ---------------------------------------------------------------------------
# NEXT row f1: one large triangular matrix across G GPUs.
#
# Top-level split of COMBRIT beta = 2: for lower T = [A 0; C B],
#   X = [A^-1 0; X21 B^-1],  X21 = -B^-1 (C A^-1).
# Phase 1: the group splits in two halves: ranks [0, G/2) invert A and ranks [G/2, G)
#          invert B, each half by this same routine on its own sub-group (recursively,
#          down to one rank: the single-GPU path), so every level of the recursion keeps
#          all G ranks busy (round 1 inverted A and B on ranks 0 and 1 only, which capped
#          the speed-up near 4.6x at G = 8).
# Phase 2: A^-1 (from rank 0) and B^-1 (from rank G/2) are broadcast.
# Phase 3: X21 is cut into 2G column panels; rank r owns panels r and 2G-1-r,
#          which balances the triangular K-ranges of C A^-1 (panel p needs
#          k >= its first column); per panel W_p = C[:, c0:] A^-1[c0:, p] and
#          X21_p = -B^-1 W_p on the DMMA engine.
# Phase 4: the panels are gathered on `dst`, which assembles X.
# Upper T = [A B12; 0 C] mirrors this with row panels of X12 = -(A^-1 B12) C^-1.
# Inputs are replicated on every rank (each rank generates / holds T).  The
# collectives are torch.distributed calls (NCCL on GPU; with gloo the tensors
# are staged through host memory, used by the CPU / single-GPU tests).
def _split_point(n):
    return 64 * ((n + 127) // 128)


def _backend_is_nccl(group):
    try:
        return dist.get_backend(group) == "nccl"
    except Exception:
        return False


def _global(group, r):
    """Global rank of group rank r (torch's src / dst arguments are global ranks)."""
    return dist.get_global_rank(group, r) if group is not None else r


def _bcast(t, src, group):
    src = _global(group, src)
    if _backend_is_nccl(group) or not t.is_cuda:
        dist.broadcast(t, src, group=group)
        return t
    h = t.cpu()
    dist.broadcast(h, src, group=group)
    t.copy_(h)
    return t


def _gather(t, dst, group):
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nccl = _backend_is_nccl(group)
    send = t if (nccl or not t.is_cuda) else t.cpu()
    out = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, out, dst=_global(group, dst), group=group)
    return out


def panel_owner_map(world):
    """Panels (2G of them) owned by each rank: r -> (r, 2G-1-r)."""
    return {r: (r, 2 * world - 1 - r) for r in range(world)}


def _int8_panels(T, uplo):
    """Whether the panel products may use the INT8 CRT engine: that opt-in engine is
    selected and the input passes its scaling guard (same decision on every rank: every
    rank holds T)."""
    from . import int8_scaling_ok, product_engine
    return product_engine() == "int8crt" and int8_scaling_ok(T, uplo)


def _panel_gemm(A, B, *, C=None, alpha=1.0, struct_a="N", struct_b="N", int8=False):
    """C = alpha A B through the INT8 CRT engine when allowed and the shape fits its
    envelope (M % 128, N % 256, K % 128, every dimension >= the engine's block threshold),
    else through the DMMA engine."""
    from . import gemm, gemm_oz, product_min_block
    M, K = A.shape
    N = B.shape[1]
    if int8 and M % 128 == 0 and N % 256 == 0 and K % 128 == 0 and min(M, N, K) >= product_min_block():
        return gemm_oz(A, B, C=C, alpha=alpha, struct_a=struct_a, struct_b=struct_b, digits=0)
    return gemm(A, B, C=C, alpha=alpha, struct_a=struct_a, struct_b=struct_b)


_SUBGROUPS = {}


def _subgroup(group, lo, hi):
    """The process group of group ranks [lo, hi) (created once per rank set; every rank of
    `group` must call this in the same order, new_group is collective)."""
    ranks = dist.get_process_group_ranks(group) if group is not None else list(range(dist.get_world_size()))
    key = tuple(ranks[lo:hi])
    if key not in _SUBGROUPS:
        _SUBGROUPS[key] = dist.new_group(list(key))
    return _SUBGROUPS[key]


def trinv_split(T, uplo="L", group=None, dst=0, inv=None, gemm=None):
    """Invert one n x n triangular matrix across the ranks of `group` (see above).

    T: the full matrix on every rank (device tensor for the GPU path).  Returns X
    on `dst` and None elsewhere.  `inv(T_block, uplo)` and `gemm(A, B, alpha,
    struct_a, struct_b)` default to this package's kernels; tests may pass CPU
    stand-ins to exercise the partition and communication logic without a GPU.
    """
    from . import trinv_lower, trinv_upper
    if inv is None:
        def inv(M, u):
            M = M.contiguous()
            return trinv_lower(M) if u == "L" else trinv_upper(M)
    if gemm is None:
        int8 = T.is_cuda and _int8_panels(T, uplo)

        def gemm(A, B, alpha, sa, sb):
            return _panel_gemm(A, B, alpha=alpha, struct_a=sa, struct_b=sb, int8=int8)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = T.shape[0]
    h = _split_point(n)
    if h >= n:  # too small to split
        X = inv(T, uplo)
        return X if rank == dst else None
    r = n - h
    src_b = world // 2 if world > 1 else 0
    # phase 1: halves of the group invert A and B, recursively (one rank: directly)
    Ainv = Binv = None
    if world > 2:
        lo, hi = _subgroup(group, 0, src_b), _subgroup(group, src_b, world)  # both created on every rank
        if rank < src_b:
            Ainv = trinv_split(T[:h, :h], uplo, group=lo, dst=0, inv=inv, gemm=gemm)
        else:
            Binv = trinv_split(T[h:, h:], uplo, group=hi, dst=0, inv=inv, gemm=gemm)
    else:
        if rank == 0:
            Ainv = inv(T[:h, :h], uplo)
        if rank == src_b:
            Binv = inv(T[h:, h:], uplo)
    if Ainv is None:
        Ainv = torch.empty((h, h), dtype=T.dtype, device=T.device)
    if Binv is None:
        Binv = torch.empty((r, r), dtype=T.dtype, device=T.device)
    # phase 2
    if world > 1:
        _bcast(Ainv, 0, group)
        _bcast(Binv, src_b, group)
    # phase 3: 2G panels of the off-diagonal block
    P = 2 * world
    w = (h + P - 1) // P
    w += w % 2  # keep 16-byte aligned column offsets
    mine = panel_owner_map(world)[rank]
    panels = []
    for p in mine:
        c0, c1 = p * w, min(h, (p + 1) * w)
        if uplo == "L":
            buf = torch.zeros((r, w), dtype=T.dtype, device=T.device)
            if c0 < c1:
                Wp = gemm(T[h:, c0:h], Ainv[c0:, c0:c1], 1.0, "N", "L")   # C A^-1, k >= c0
                buf[:, : c1 - c0] = gemm(Binv, Wp, -1.0, "L", "N")        # -B^-1 W
        else:
            buf = torch.zeros((w, r), dtype=T.dtype, device=T.device)
            if c0 < c1:
                Wp = gemm(Ainv[c0:c1, c0:], T[c0:h, h:], 1.0, "U", "N")   # A^-1 B12, k >= c0
                buf[: c1 - c0, :] = gemm(Wp, Binv, -1.0, "N", "U")        # -W C^-1
        panels.append(buf)
    # phase 4
    stack = torch.stack(panels)
    got = _gather(stack, dst, group) if world > 1 else [stack]
    if rank != dst:
        return None
    X = torch.zeros((n, n), dtype=T.dtype, device=T.device)
    X[:h, :h] = Ainv
    X[h:, h:] = Binv
    for rk, part in enumerate(got):
        part = part.to(T.device)
        for k, p in enumerate(panel_owner_map(world)[rk]):
            c0, c1 = p * w, min(h, (p + 1) * w)
            if c0 >= c1:
                continue
            if uplo == "L":
                X[h:, c0:c1] = part[k][:, : c1 - c0]
            else:
                X[c0:c1, h:] = part[k][: c1 - c0, :]
    return X


# ---------------------------------------------------------------------------
# f1 with peer-memory transport: the broadcast and the gather of trinv_split
# fused into the kernels.  `dst` owns X; every rank maps it through CUDA IPC
# (NVLink peer memory on a multi-GPU node).  Phase 1 writes A^-1 and B^-1 straight
# into X on `dst`; phase 3 reads them from there as TMA operands of the panel
# products (P2P loads replace the broadcast) and the epilogue of the second product
# stores each X21 panel straight into X on `dst` (P2P stores replace the gather).
# The only collectives left are two barriers (phase ordering); no data moves
# through NCCL.  Requires an even n and a device tensor T (TMA operand layout).
def _share_from(t, src, group):
    """A view of rank `src`'s CUDA tensor `t` on every rank (CUDA IPC handle via the process group)."""
    from torch.multiprocessing.reductions import reduce_tensor
    rank = dist.get_rank(group)
    obj = [reduce_tensor(t) if rank == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    if rank == src:
        return t
    fn, args = obj[0]
    return fn(*args)


def trinv_split_p2p(T, uplo="L", group=None, dst=0):
    """trinv_split with the data exchange done by the kernels over peer memory (see above)."""
    from . import trinv_lower, trinv_upper
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = T.shape[0]
    h = _split_point(n)
    if world == 1 or h >= n or n % 2:
        return trinv_split(T, uplo, group=group, dst=dst)
    r = n - h
    inv = trinv_lower if uplo == "L" else trinv_upper
    Xown = torch.zeros((n, n), dtype=T.dtype, device=T.device) if rank == dst else None
    X = _share_from(Xown, dst, group)
    src_b = min(1, world - 1)
    # phase 1: diagonal-block inverses written straight into X on dst
    if rank == 0:
        inv(T[:h, :h], out=X[:h, :h])
    if rank == src_b:
        inv(T[h:, h:], out=X[h:, h:])
    torch.cuda.synchronize()
    dist.barrier(group=group)
    # phase 3: 2G balanced panels; operands read from X on dst, results stored there
    int8 = _int8_panels(T, uplo)

    def _gemm(A, B, C=None, alpha=1.0, struct_a="N", struct_b="N"):
        return _panel_gemm(A, B, C=C, alpha=alpha, struct_a=struct_a, struct_b=struct_b, int8=int8)
    P = 2 * world
    w = (h + P - 1) // P
    w += w % 2
    for p in panel_owner_map(world)[rank]:
        c0, c1 = p * w, min(h, (p + 1) * w)
        if c0 >= c1:
            continue
        if uplo == "L":
            Wp = _gemm(T[h:, c0:h], X[c0:h, c0:c1], struct_b="L")             # C A^-1, k >= c0
            _gemm(X[h:, h:], Wp, C=X[h:, c0:c1], alpha=-1.0, struct_a="L")    # -B^-1 W -> X on dst
        else:
            Wp = _gemm(X[c0:c1, c0:h], T[c0:h, h:], struct_a="U")             # A^-1 B12, k >= c0
            _gemm(Wp, X[h:, h:], C=X[c0:c1, h:], alpha=-1.0, struct_b="U")    # -W C^-1 -> X on dst
    torch.cuda.synchronize()
    dist.barrier(group=group)
    return Xown if rank == dst else None

