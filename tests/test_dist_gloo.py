"""Multi-process (world_size 2-3, gloo, CPU) tests of the sharding / reduction / halo
exchange logic used by bench.py under torchrun and by multi-rank
deployments holding per-rank buffer ranges.  The same code runs over NCCL on B200s."""
import os
import socket

import pytest

from paper_2108_07004_b200.sharding import rank_batches, shard_range, sum_counts


def test_shard_range_partitions():
    for n in (1, 7, 16, 4096):
        for w in (1, 2, 3, 8):
            got = []
            for r in range(w):
                lo, hi = shard_range(n, w, r)
                got += list(range(lo, hi))
            assert got == list(range(n))


def test_rank_batches_shard_the_stream():
    """bench.py's plan (sharding.rank_batches): the C5 stream of 4096 buffers, 128 per batch.
    weak: every rank's batches lie in its own contiguous shard, consecutive in stream order,
    and no two ranks ever process the same buffer; strong: one step covers the whole stream
    exactly once over all ranks, for any world size (including ragged shards)."""
    for S, B in ((4096, 128), (100, 7), (13, 5)):
        for w in (1, 2, 3, 4, 8):
            seen = set()
            for r in range(w):
                lo, hi = shard_range(S, w, r)
                mine = []
                for s in range(5):
                    for b0, cnt in rank_batches(s, r, w, B, S, "weak"):
                        assert lo <= b0 and b0 + cnt <= hi and 0 < cnt <= B
                        mine += list(range(b0, b0 + cnt))
                if 5 * B <= hi - lo:  # no wrap inside the shard: the batches walk it in order
                    assert mine == list(range(lo, lo + 5 * B))
                assert not (set(mine) & seen)
                seen |= set(mine)
            strong = [b for r in range(w) for b0, cnt in rank_batches(0, r, w, B, S, "strong")
                      for b in range(b0, b0 + cnt)]
            assert sorted(strong) == list(range(S))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2108_07004_b200.sharding import reduce_counts
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(10, world, rank)
    # fake per-buffer counters: buffer b has b bit errors, flags only on buffer 7
    per = [dict(bit_errors=b, sym_errors=b // 2, bits=100, symbols=25, clipped_samples=0, gated_updates=1,
                flags=1 if b == 7 else 0) for b in range(lo, hi)]
    tot, tmax = reduce_counts(sum_counts(per), 10.0 + rank)
    q.put((rank, tot, tmax))
    dist.destroy_process_group()


def test_gloo_world2_reduction():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tot, tmax in res:
        assert tot["bit_errors"] == sum(range(10))
        assert tot["sym_errors"] == sum(b // 2 for b in range(10))
        assert tot["bits"] == 1000 and tot["symbols"] == 250
        assert tot["flags"] == 1
        assert tmax == 11.0
    assert torch is not None


def _halo_worker(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2108_07004_b200.sharding import exchange_halos, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, nbuf, left, right = 1024, 6, 300, 80
    rng = np.random.default_rng(5)
    glob = torch.from_numpy(rng.integers(-2048, 2048, left + nbuf * N + right).astype(np.int16))
    lo, hi = shard_range(nbuf, world, rank)
    mine = glob[lo * N: hi * N + left + right].clone()  # [left | own | right] window of the global stream
    want = mine.clone()
    if rank > 0:
        mine[:left] = 0          # halos that live on the neighbours
    if rank + 1 < world:
        mine[-right:] = 0
    exchange_halos(mine, left, right)
    q.put((rank, bool(torch.equal(mine, want))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_exchange(world):
    """exchange_halos fills every inner rank boundary with the neighbours' samples
    (SURVEY 8(e) optional P2P halo exchange), world sizes 2 and 3 over gloo."""
    pytest.importorskip("torch")
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def _fake_counts(b, pool=64):
    """per-buffer counters of stream buffer b (a function of its pool buffer, as in the bench)"""
    p = b % pool
    return dict(bit_errors=3 * p + 1, sym_errors=p, bits=1 << 21, symbols=1 << 20, clipped_samples=p % 3,
                gated_updates=7 * p, flags=2 if p == 5 else 0)


def _plan_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2108_07004_b200.sharding import rank_batches, reduce_counts, sum_counts
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    per = [_fake_counts(b) for b0, cnt in rank_batches(0, rank, world, 128, 4096, "strong")
           for b in range(b0, b0 + cnt)]
    tot, tmax = reduce_counts(sum_counts(per), 5.0 * (rank + 1))
    q.put((rank, tot, tmax))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_stream_totals_equal_single_rank(world):
    """The functions bench.py calls under torchrun (rank_batches -> per-buffer counters ->
    sum_counts -> reduce_counts over the process group), at world sizes 2 and 3 over gloo:
    the reduced totals of one strong-scaling pass over the 4096-buffer C5 stream equal the
    single-rank totals, and the time is the max over ranks."""
    pytest.importorskip("torch")
    import torch.multiprocessing as tmp
    single = sum_counts([_fake_counts(b) for b0, cnt in rank_batches(0, 0, 1, 128, 4096, "strong")
                         for b in range(b0, b0 + cnt)])
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tot, tmax in res:
        assert tot == single, (tot, single)
        assert tmax == 5.0 * world
