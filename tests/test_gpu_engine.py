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

from engine_workload import CASES, SHAPE, HashTokens  # noqa: E402

pytestmark = pytest.mark.gpu

import paper_2410_00161_b200 as K  # noqa: E402

GOLDEN = {c["name"]: c["records"] for c in json.load(open(os.path.join(HERE, "golden", "engine_cases.json")))}


@pytest.mark.parametrize("name,kw,reqs", CASES, ids=[c[0] for c in CASES])
def test_engine_matches_reference(name, kw, reqs):
    cfg = K.AttentionConfig(SHAPE["n_q"], SHAPE["n_k"], SHAPE["d"], SHAPE["layers"])
    eng = K.Engine(cfg, K.MetricConfig(), K.POLICY_PRESETS[kw["policy"]], kw["num_blocks"], SHAPE["block_size"],
                   rate=kw["rate"], budget_floor=kw["budget_floor"], record_schedules=True)
    for i, (pl, ot) in enumerate(reqs):
        eng.submit(HashTokens(1000 + i, pl, ot, SHAPE["layers"], SHAPE["n_q"], SHAPE["n_k"], SHAPE["d"]))
    got = [r.to_dict() for r in eng.run_to_completion()]
    want = GOLDEN[name]
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g == w, (name, g["step"])
