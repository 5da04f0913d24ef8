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
