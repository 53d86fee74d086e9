"""Multi-GPU plumbing: buffer sharding and counter reduction.

The KK chain shards buffer-by-buffer: the outputs of buffer b depend only on the
raw window [bN - left, (b+1)N + right) (adaptive taps restart per sub-block,
reading R10; the tone phase is buffer-local, reading R7), so ranks process
disjoint buffer ranges.  The collectives: one all_reduce(SUM) of the int64 error
counters (and MAX of elapsed time) at the end of a run or report window, and -- when
each rank holds only its own buffers -- one neighbour halo exchange per contiguous range
(`exchange_halos`, ~35 KB per side for K = 4096): torch.distributed over NCCL on B200s,
gloo in the CPU tests.
"""
from __future__ import annotations

COUNT_KEYS = ("bit_errors", "sym_errors", "bits", "symbols", "clipped_samples", "gated_updates")


def shard_range(n_buffers: int, world: int, rank: int):
    """Contiguous buffer range [lo, hi) of `rank` (sizes differ by at most 1)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(int(n_buffers), int(world))
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def weak_step_buffers(step: int, rank: int, world: int, batch: int, pool: int):
    """First pool buffer of `rank`'s batch in `step` for a weak-scaling run that
    cycles a pool of distinct buffers (each rank a different batch per step)."""
    return (rank * batch + step * batch * world) % pool


def sum_counts(per_buffer):
    tot = {k: 0 for k in COUNT_KEYS}
    flags = 0
    for c in per_buffer:
        for k in COUNT_KEYS:
            tot[k] += int(c[k])
        flags |= int(c.get("flags", 0))
    tot["flags"] = flags
    return tot


def reduce_counts(local: dict, elapsed_ms: float, device=None, group=None):
    """all_reduce(SUM) of the counters and all_reduce(MAX) of the elapsed time."""
    import torch
    import torch.distributed as dist

    v = torch.tensor([int(local[k]) for k in COUNT_KEYS] + [int(local.get("flags", 0))], dtype=torch.int64,
                     device=device)
    t = torch.tensor([float(elapsed_ms)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        flags = v[-1:].clone()
        dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
        v[-1] = flags[0]
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    out = {k: int(v[i]) for i, k in enumerate(COUNT_KEYS)}
    out["flags"] = int(v[-1])
    return out, float(t.item())


def exchange_halos(stream, left: int, right: int, group=None):
    """Halo exchange between neighbouring ranks ("the first buffer's left
    halo and the last buffer's right halo can be P2P-exchanged over NVLink").

    stream: this rank's 1-D int16 tensor laid out as [left halo | own buffers | right halo]
    (contiguous buffer ranges per rank, `shard_range`).  Rank r's left halo is the last
    `left` own samples of rank r-1 and its right halo the first `right` own samples of
    rank r+1; both are exchanged with one batch of point-to-point sends/receives (NCCL
    over NVLink for CUDA tensors, gloo for CPU tensors).  The outer ranks keep the halos
    they were given (the stream's guard data).  Each rank needs at least max(left, right)
    own samples.  In place; returns `stream`."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return stream
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = stream.numel()
    own_lo, own_hi = left, n - right
    if own_hi - own_lo < max(left, right):
        raise ValueError("each rank needs at least max(left, right) own samples")
    peer = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    ops = []
    if rank + 1 < world:
        ops.append(dist.P2POp(dist.isend, stream[own_hi - left:own_hi].contiguous(), peer(rank + 1), group))
        ops.append(dist.P2POp(dist.irecv, stream[own_hi:], peer(rank + 1), group))
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, stream[own_lo:own_lo + right].contiguous(), peer(rank - 1), group))
        ops.append(dist.P2POp(dist.irecv, stream[:own_lo], peer(rank - 1), group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return stream
