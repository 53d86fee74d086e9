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

import numpy as np

COUNT_KEYS = ("bit_errors", "sym_errors", "bits", "symbols", "clipped_samples", "gated_updates")


def shard_range(n_buffers: int, world: int, rank: int):
    """Contiguous buffer range [lo, hi) of `rank` (sizes differ by at most 1)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(int(n_buffers), int(world))
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def rank_batches(step: int, rank: int, world: int, batch: int, n_stream: int, scaling: str = "weak"):
    """The batches (first stream buffer, buffer count) `rank` submits in `step` when a
    continuous stream of `n_stream` buffers (C5: 4096) is sharded contiguously over `world`
    ranks (rank r owns shard_range(n_stream, world, r)).

    weak   -- per-GPU work fixed: one batch of up to `batch` consecutive buffers per step,
              walking the rank's own range in stream order (and wrapping inside it);
              batches never cross the range end, so ranks never process the same buffer.
    strong -- total work fixed: a step is one pass over the WHOLE stream, i.e. the rank's
              range in consecutive batches of up to `batch` buffers."""
    lo, hi = shard_range(n_stream, world, rank)
    n = hi - lo
    if n <= 0 or batch <= 0:
        return []
    if scaling == "strong":
        return [(b, min(batch, hi - b)) for b in range(lo, hi, batch)]
    if scaling != "weak":
        raise ValueError(scaling)
    start = lo + (step * batch) % n
    return [(start, min(batch, hi - start))]


def max_over_ranks(value: float, device=None, group=None) -> float:
    """all_reduce(MAX) of a per-rank time (the bench's max-over-ranks timing rule)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def comm_info(group=None) -> dict:
    """The process group the counters are reduced over (logged in the bench line)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return {"backend": None, "world": 1}
    info = {"backend": str(dist.get_backend(group)), "world": dist.get_world_size(group)}
    if info["backend"] == "nccl":
        try:
            info["nccl_version"] = ".".join(str(x) for x in torch.cuda.nccl.version())
        except Exception:
            pass
    return info


def sum_counts(per_buffer):
    """Sum per-buffer counter dicts (or a structured counter array) into one dict."""
    if hasattr(per_buffer, "dtype") and getattr(per_buffer.dtype, "names", None):
        tot = {k: int(per_buffer[k].sum()) for k in COUNT_KEYS}
        tot["flags"] = int(np.bitwise_or.reduce(per_buffer["flags"])) if len(per_buffer) else 0
        return tot
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
