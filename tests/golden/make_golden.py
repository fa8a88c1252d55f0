"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
records, for seeded random inputs, the reference's own outputs:

* ``compress_cases.json`` - full compression rounds (pagedkv.compression.
  compress): initial per-slot state + tables, the CompressionSchedule.to_dict
  payload, and the final state;
* ``decode_cases.json`` - paged_attention outputs/rows + accumulate_decode;
* ``metric_cases.json`` - gqa_attention -> window_metrics / full_metrics;
* ``alloc_cases.json`` - BlockManager allocate/free traces.

The committed JSON files are small; tests compare the oracle (and, on the
GPU, the CUDA path) against them.  Floats are stored with repr precision so
they round-trip exactly.
"""

from __future__ import annotations

import base64
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from pagedkv.attention import AttentionConfig, gqa_attention, paged_attention  # noqa: E402
from pagedkv.block_manager import BlockManager  # noqa: E402
from pagedkv.cache import BlockTables, UnifiedKVCache, append_kv  # noqa: E402
from pagedkv.compression import compress  # noqa: E402
from pagedkv.errors import PreemptionNeeded  # noqa: E402
from pagedkv.metrics import (  # noqa: E402
    MetricConfig,
    MetricsStore,
    accumulate_decode,
    full_metrics,
    window_metrics,
)

OUT = os.path.dirname(os.path.abspath(__file__))


def rig(num_blocks, b, d, layers, heads):
    cache = UnifiedKVCache(num_blocks, b, d)
    tables = BlockTables(layers, heads, b)
    manager = BlockManager(num_blocks, tables)
    store = MetricsStore(num_blocks, b)
    return cache, tables, manager, store


def fill(cache, tables, manager, store, seq, layer, head, metrics, rng, protected=None):
    """Populate a head with len(metrics) KVs through the reference API."""
    b = tables.block_size
    for _ in range(-(-len(metrics) // b)):
        manager._take(seq, layer, head)
    for i, m in enumerate(metrics):
        handle = append_kv(tables, cache, seq, layer, head,
                           rng.standard_normal(cache.head_dim),
                           rng.standard_normal(cache.head_dim))
        store.on_append(handle, logical=i)
        store.metrics[handle.block, handle.offset] = m
        if protected is not None and protected[i]:
            store.protected[handle.block, handle.offset] = True


def enc(arr):
    """float64/int64 array -> compact base64 record (decoded by tests/golden_io.py)."""
    arr = np.ascontiguousarray(arr)
    return {"dtype": str(arr.dtype), "shape": list(arr.shape),
            "b64": base64.b64encode(arr.tobytes()).decode()}


def snapshot(cache, tables, manager, store, blocks=None, with_kv=False):
    """Per-slot state restricted to `blocks` (default: every owned block)."""
    seqs = tables.sequences
    if blocks is None:
        blocks = sorted(b for s in seqs for b in tables.owned_blocks(s))
    bsz = tables.block_size
    flats = (np.asarray(blocks, dtype=np.int64)[:, None] * bsz + np.arange(bsz)).reshape(-1)
    snap = {
        "blocks": list(map(int, blocks)),
        "metric": enc(store.metrics_flat[flats]),
        "logical": enc(store.logical_flat[flats]),
        "protected": store.protected_flat[flats].astype(int).tolist(),
        "fresh": store.fresh_flat[flats].astype(int).tolist(),
        "free": sorted(manager._free_set),
        "tables": {str(s): [[list(tables.blocks(s, m, h)) for h in range(tables.num_kv_heads)]
                            for m in range(tables.num_layers)] for s in seqs},
        "ctx": {str(s): [[tables.context_len(s, m, h) for h in range(tables.num_kv_heads)]
                         for m in range(tables.num_layers)] for s in seqs},
    }
    if with_kv:
        snap["keys"] = enc(cache.keys_flat[flats])
        snap["values"] = enc(cache.values_flat[flats])
    return snap


def tie_metrics(rng, n):
    """Metric lists with heavy ties (pooled-metric-like) or i.i.d. values."""
    kind = rng.integers(0, 3)
    if kind == 0:
        return list(rng.random(n))
    if kind == 1:
        return list(np.round(rng.random(n), 1))
    base = rng.random(max(1, n // 3 + 1))
    return [float(base[i // 3]) for i in range(n)]


def make_compress_cases():
    rng = np.random.default_rng(20241001)
    cases = []
    for case in range(60):
        b = int(rng.choice([2, 4, 16]))
        layers = int(rng.integers(1, 3))
        heads = int(rng.integers(1, 4))
        nseq = int(rng.integers(1, 3))
        d = 4
        cache, tables, manager, store = rig(160, b, d, layers, heads)
        budgets = {}
        for s in range(nseq):
            sid = int(rng.integers(0, 50)) * 2 + s  # arbitrary distinct ids
            while tables.has_sequence(sid):
                sid += 1
            tables.add_sequence(sid)
            for m in range(layers):
                for h in range(heads):
                    n = int(rng.integers(1, 6 * b))
                    prot = rng.random(n) < 0.1 if rng.random() < 0.3 else None
                    fill(cache, tables, manager, store, sid, m, h, tie_metrics(rng, n), rng, prot)
                    if rng.random() < 0.2:
                        # a couple of fresh slots
                        flats = tables.head_slots_flat(sid, m, h)[: tables.context_len(sid, m, h)]
                        store.fresh_flat[flats[-1]] = True
            budgets[sid] = int(rng.integers(0, 3 * layers * heads + 2))
        before = snapshot(cache, tables, manager, store, with_kv=True)
        schedule = compress(cache, tables, manager, store, budgets)
        after = snapshot(cache, tables, manager, store, blocks=before["blocks"], with_kv=True)
        cases.append({
            "num_blocks": 160, "block_size": b, "head_dim": d, "layers": layers,
            "heads": heads, "budgets": [[k, v] for k, v in budgets.items()],
            "before": before, "schedule": schedule.to_dict(), "after": after,
        })
    return cases


def make_decode_cases():
    rng = np.random.default_rng(77)
    cases = []
    for _ in range(24):
        b = int(rng.choice([2, 4, 16]))
        heads = int(rng.choice([1, 2, 4]))
        r = int(rng.integers(1, 5))
        d = int(rng.choice([4, 8, 16, 32]))
        layers = 2
        cache, tables, manager, store = rig(128, b, d, layers, heads)
        tables.add_sequence(3)
        for m in range(layers):
            for h in range(heads):
                fill(cache, tables, manager, store, 3, m, h, list(rng.random(int(rng.integers(1, 48)))), rng)
        cfg = AttentionConfig(heads * r, heads, d, layers)
        layer = int(rng.integers(0, layers))
        q = rng.standard_normal((heads * r, d))
        before = snapshot(cache, tables, manager, store, with_kv=True)
        out, rows = paged_attention(q, cache, tables, 3, layer, cfg)
        agg = "L2" if rng.random() < 0.5 else "L1"
        accumulate_decode(store, tables, 3, layer, rows, MetricConfig(mode="full", aggregation=agg))
        cases.append({
            "block_size": b, "heads": heads, "r": r, "head_dim": d, "layers": layers,
            "num_blocks": 128, "layer": layer, "aggregation": agg, "seq": 3,
            "query": enc(q), "before": before, "out": enc(out),
            "rows": [enc(row) for row in rows],
            "metric_after": enc(store.metrics_flat[
                (np.asarray(before["blocks"])[:, None] * b + np.arange(b)).reshape(-1)]),
        })
    return cases


def make_metric_cases():
    rng = np.random.default_rng(5150)
    cases = []
    for _ in range(24):
        heads = int(rng.choice([1, 2, 4]))
        r = int(rng.integers(1, 5))
        L = int(rng.integers(1, 80))
        d = int(rng.choice([4, 8, 16]))
        q = rng.standard_normal((heads * r, L, d))
        k = rng.standard_normal((heads, L, d))
        v = rng.standard_normal((heads, L, d))
        _, attn = gqa_attention(q, k, v, AttentionConfig(heads * r, heads, d, 1))
        agg = "L2" if rng.random() < 0.6 else "L1"
        window = int(rng.integers(1, 12))
        pool = int(rng.choice([1, 3, 7]))
        wcfg = MetricConfig(mode="window", aggregation=agg, window=window, pool=pool)
        wm, prot = window_metrics(attn, wcfg, heads)
        excl = int(rng.integers(0, 12))
        fm = full_metrics(attn, MetricConfig(mode="full", aggregation=agg, excluded=excl), heads)
        cases.append({
            "heads": heads, "r": r, "L": L, "d": d, "aggregation": agg,
            "window": window, "pool": pool, "excluded": excl,
            "q": enc(q), "k": enc(k),
            "window_metrics": enc(wm), "protected": prot.astype(int).tolist(),
            "full_metrics": enc(fm),
        })
    return cases


def make_alloc_cases():
    rng = np.random.default_rng(99)
    cases = []
    for _ in range(20):
        b = int(rng.choice([2, 4, 16]))
        layers = int(rng.integers(1, 3))
        heads = int(rng.integers(1, 3))
        num_blocks = int(rng.integers(16, 200))
        tables = BlockTables(layers, heads, b)
        manager = BlockManager(num_blocks, tables)
        ops = []
        live = []
        next_id = 0
        for _ in range(40):
            x = rng.random()
            if x < 0.4 or not live:
                tokens = int(rng.integers(1, 5 * b))
                try:
                    manager.allocate_prefill(next_id, tokens)
                    for m, h in tables.heads(next_id):
                        tables.set_context_len(next_id, m, h, tokens)
                    ops.append({"op": "prefill", "seq": next_id, "tokens": tokens, "ok": True})
                    live.append(next_id)
                except PreemptionNeeded as exc:
                    ops.append({"op": "prefill", "seq": next_id, "tokens": tokens,
                                "ok": False, "shortfall": exc.shortfall})
                next_id += 1
            elif x < 0.8:
                # grow every head by a random number of tokens, one decode step each
                steps = int(rng.integers(1, b + 2))
                for _ in range(steps):
                    try:
                        counts = manager.allocate_decode_step(list(live))
                        for s in live:
                            for m, h in tables.heads(s):
                                tables.set_context_len(s, m, h, tables.context_len(s, m, h) + 1)
                        ops.append({"op": "decode", "seqs": list(live), "ok": True,
                                    "counts": [[k, v] for k, v in counts.items()],
                                    "tables": {str(s): [[list(tables.blocks(s, m, h)) for h in range(heads)]
                                                        for m in range(layers)] for s in tables.sequences},
                                    "free_count": manager.free_count})
                    except PreemptionNeeded as exc:
                        ops.append({"op": "decode", "seqs": list(live), "ok": False,
                                    "shortfall": exc.shortfall})
                        break
            else:
                victim = live.pop(int(rng.integers(0, len(live))))
                freed = manager.free_sequence(victim)
                ops.append({"op": "free_sequence", "seq": victim, "freed": freed})
            for op in ops:
                if "tables" not in op:
                    op["tables"] = {str(s): [[list(tables.blocks(s, m, h)) for h in range(heads)]
                                             for m in range(layers)] for s in tables.sequences}
                    op["free_count"] = manager.free_count
        cases.append({"block_size": b, "layers": layers, "heads": heads,
                      "num_blocks": num_blocks, "ops": ops})
    return cases


def main():
    for name, fn in (
        ("compress_cases.json", make_compress_cases),
        ("decode_cases.json", make_decode_cases),
        ("metric_cases.json", make_metric_cases),
        ("alloc_cases.json", make_alloc_cases),
    ):
        data = fn()
        with open(os.path.join(OUT, name), "w") as fh:
            json.dump(data, fh, separators=(",", ":"))
        print(name, len(data), os.path.getsize(os.path.join(OUT, name)))


if __name__ == "__main__":
    main()
