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
    got = gather_counts([len(mine), sum(mine), rank * 7, 3]).tolist()
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


class _StubEngine:
    """Duck-typed local engine: request j finishes after `steps` decode steps;
    free pool = 100 - live requests."""

    def __init__(self):
        self.waiting, self.running, self.step_index = [], [], 0

        class M:
            free_count = 100
        self.manager = M()

    def submit(self, src):
        self.waiting.append(src)

    @property
    def active(self):
        return bool(self.waiting or self.running)

    def step(self):
        from paper_2410_00161_b200.engine import StepRecord
        self.step_index += 1
        rec = StepRecord(step=self.step_index)
        if self.waiting:
            self.running.append([self.waiting.pop(0), 0])
            rec.admitted = 1
        for r in self.running:
            r[1] += 1
        rec.batch_size = len(self.running)
        done = [r for r in self.running if r[1] >= r[0]]
        for r in done:
            self.running.remove(r)
        rec.finished = len(done)
        rec.free_blocks = self.manager.free_count - len(self.running)
        return rec


def _engine_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2410_00161_b200.sharding import ShardedEngine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    se = ShardedEngine(_StubEngine())
    for steps in [3, 1, 4, 1, 5, 9, 2]:  # request i -> rank i % 2
        se.submit(steps)
    local, glob = se.run_to_completion()
    q.put((rank, se.owned, [r.step for r in local], [g.totals for g in glob], [g.per_rank for g in glob]))
    dist.destroy_process_group()


def test_sharded_engine_lock_step_two_ranks():
    """Lock-step across ranks with unequal work: the idle rank keeps joining
    the gathers, totals are per-step sums over ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_engine_worker, args=(r, 2, 29519, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, own0, steps0, tot0, per0), (_, own1, steps1, tot1, per1) = res
    assert own0 == [0, 2, 4, 6] and own1 == [1, 3, 5]
    assert tot0 == tot1 and per0 == per1
    assert len(tot0) == max(len(steps0), len(steps1))
    # rank 0: requests of 3, 4, 5, 2 steps admitted one per step
    assert steps0 == list(range(1, len(steps0) + 1))
    for t, g in enumerate(tot0):
        assert g["admitted"] == sum(p["admitted"] for p in per0[t])
        assert g["free_blocks"] == sum(p["free_blocks"] for p in per0[t])
    assert sum(g["admitted"] for g in tot0) == 7
    assert sum(g["finished"] for g in tot0) == 7
