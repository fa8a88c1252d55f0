"""World-size-2 gloo test of the multi-GPU host logic (CPU only)."""

from __future__ import annotations

import os

import pytest
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2410_00161_b200.sharding import gather_counts, shard_sequences

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_sequences(list(range(10)), rank, world)
    got = gather_counts([len(mine), sum(mine), rank * 7, 3])
    q.put((rank, mine, got))
    dist.destroy_process_group()


def test_sharding_and_count_gather_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29517
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, m0, g0), (_, m1, g1) = res
    assert m0 == [0, 2, 4, 6, 8] and m1 == [1, 3, 5, 7, 9]
    assert sorted(m0 + m1) == list(range(10))
    assert g0 == g1 == [[5, 20, 0, 3], [5, 25, 7, 3]]
