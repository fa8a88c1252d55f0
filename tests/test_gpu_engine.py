"""Device Engine vs the reference Engine's StepRecords on the
same deterministic workloads (GPU).

Golden records come from running pkg/src/pagedkv/engine.py itself
(tests/golden/make_engine_golden.py).  Token activations are bf16-exact, so
the caches hold identical K/V; metrics differ only by fp32-vs-f64 rounding.
Counters (admissions, batch sizes, compressions, freed blocks, evicted KVs,
preemptions, finished, free blocks, fragmentation) and the full per-round
schedule records (per-head evictions, freed ids, move lists) must match."""

from __future__ import annotations

import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from engine_workload import CASES, SHAPE, SHARD_WORLD, HashTokens, make_policy, shard  # noqa: E402

pytestmark = pytest.mark.gpu

import paper_2410_00161_b200 as K  # noqa: E402

CASES_JSON = json.load(open(os.path.join(HERE, "golden", "engine_cases.json")))
GOLDEN = {c["name"]: c["records"] for c in CASES_JSON}
GOLDEN_SHARDS = {c["name"]: c["shards"] for c in CASES_JSON}


@pytest.mark.parametrize("graph_after", [0, None], ids=["graph-every-step", "graph-stable-batches"])
@pytest.mark.parametrize("name,kw,reqs", CASES, ids=[c[0] for c in CASES])
def test_engine_matches_reference(name, kw, reqs, graph_after):
    """graph_after=0: every decode step replays a CUDA graph (captured anew
    whenever the batch changes); None: the default (graphs for batches
    stable for a few steps, eager otherwise)."""
    cfg = K.AttentionConfig(SHAPE["n_q"], SHAPE["n_k"], SHAPE["d"], SHAPE["layers"])
    extra = {} if graph_after is None else {"graph_after": graph_after}
    eng = K.Engine(cfg, K.MetricConfig(), make_policy(K, kw["policy"]), kw["num_blocks"], SHAPE["block_size"],
                   rate=kw["rate"], budget_floor=kw["budget_floor"], record_schedules=True, **extra)
    for i, (pl, ot) in enumerate(reqs):
        eng.submit(HashTokens(1000 + i, pl, ot, SHAPE["layers"], SHAPE["n_q"], SHAPE["n_k"], SHAPE["d"]))
    got = [r.to_dict() for r in eng.run_to_completion()]
    want = GOLDEN[name]
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g == w, (name, g["step"])


def _shard_worker(rank, world, port, name, kw, reqs, q):
    """One rank of a 2-rank job sharing cuda:0 (the box has one GPU): its own
    Engine and device pool, gloo for the counter all-gather."""
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = K.AttentionConfig(SHAPE["n_q"], SHAPE["n_k"], SHAPE["d"], SHAPE["layers"])
        eng = K.Engine(cfg, K.MetricConfig(), make_policy(K, kw["policy"]), kw["num_blocks"], SHAPE["block_size"],
                       rate=kw["rate"], budget_floor=kw["budget_floor"], record_schedules=True, device="cuda:0")
        se = K.ShardedEngine(eng)
        for i, (pl, ot) in enumerate(reqs):
            se.submit(HashTokens(1000 + i, pl, ot, SHAPE["layers"], SHAPE["n_q"], SHAPE["n_k"], SHAPE["d"]))
        local, glob = se.run_to_completion()
        q.put((rank, [r.to_dict() for r in local], [g.totals for g in glob], se.owned))
    except Exception as exc:  # surface the failure in the parent
        q.put((rank, repr(exc), None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [c for c in CASES if c[0] in ("prefill-preempt", "decode-compress-then-preempt",
                                                               "kv-limit")], ids=lambda c: c[0])
def test_sharded_engine_two_ranks_match_reference_shards(case):
    """Sequences sharded over 2 ranks: each rank's records equal the
    reference engine run on the requests that rank owns (per-rank oracle,
    bit-exact schedules), and the gathered totals are the per-step sums."""
    import torch.multiprocessing as mp

    name, kw, reqs = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + sum(map(ord, name)) % 200
    procs = [ctx.Process(target=_shard_worker, args=(r, SHARD_WORLD, port, name, kw, reqs, q))
             for r in range(SHARD_WORLD)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
    for rank, local, glob, owned in res:
        assert glob is not None, local
        assert owned == [i for i, _ in shard(reqs, rank)]
        assert local == GOLDEN_SHARDS[name][rank], (name, rank)
    for p in procs:
        assert p.exitcode == 0
    # gathered totals: the sum over ranks of each rank's record at that step
    glob = res[0][2]
    assert res[1][2] == glob
    n = max(len(g) for g in GOLDEN_SHARDS[name])
    assert len(glob) == n
    for t in range(n):
        for f in ("admitted", "batch_size", "compressions", "blocks_freed", "kvs_evicted", "preemptions", "finished"):
            want = sum(g[t][f] for g in GOLDEN_SHARDS[name] if t < len(g))
            assert glob[t][f] == want, (t, f)
