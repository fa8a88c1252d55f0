"""K1 paged decode + K0 allocator parity against the CPU oracle (GPU).

Tolerances (bf16 KV and queries are fed to BOTH sides, so the only
difference is fp32 accumulation + exp2 in the kernel vs float64 in the
oracle): outputs and attention rows 2e-3 absolute, metrics 1e-3 relative.
Integer state (tables, ctx, logical, flags, free pool) must match exactly.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_io import dec, load
from gpu_rig import DevRig, as_np, bf16_round, random_state
from oracle import kvc_oracle as O
from oracle_rig import state_from_snapshot

pytestmark = pytest.mark.gpu

import paper_2410_00161_b200 as K  # noqa: E402
from paper_2410_00161_b200 import errors as E  # noqa: E402

ATOL = 2e-3  # attention rows (fp32 scores)
OUT_ATOL = 1e-2  # outputs: P enters the P.V tensor-core product in bf16 (as FlashAttention)
MET_RTOL = 1e-3


def assert_same_ints(st_dev, st_ref):
    assert {s: t for s, t in st_dev.tables.items()} == {s: t for s, t in st_ref.tables.items()}
    for s in st_ref.ctx:
        assert np.array_equal(st_dev.ctx[s], st_ref.ctx[s])
    assert np.array_equal(st_dev.free, st_ref.free)
    assert np.array_equal(st_dev.logical, st_ref.logical)
    assert np.array_equal(st_dev.protected, st_ref.protected)
    assert np.array_equal(st_dev.fresh, st_ref.fresh)


def test_library_loads_with_every_symbol():
    from paper_2410_00161_b200 import _lib

    lib = _lib.load()
    assert lib.kvc_abi_version() == 3
    for name in _lib.EXPORTED:
        assert hasattr(lib, name)


@pytest.mark.parametrize("i", range(len(load("alloc_cases.json"))))
def test_allocator_matches_reference_trace(i):
    """Replay the reference BlockManager traces on the device allocator."""
    case = load("alloc_cases.json")[i]
    rig = DevRig(case["num_blocks"], case["block_size"], 8, case["layers"], case["heads"], max_seqs=64)
    t, mgr = rig.tables, rig.manager
    for op in case["ops"]:
        if op["op"] == "prefill":
            try:
                mgr.allocate_prefill(op["seq"], op["tokens"])
                for m, h in t.heads(op["seq"]):
                    t.set_context_len(op["seq"], m, h, op["tokens"])
                assert op["ok"]
            except E.PreemptionNeeded as exc:
                assert not op["ok"] and exc.shortfall == op["shortfall"]
        elif op["op"] == "decode":
            try:
                counts = mgr.allocate_decode_step(op["seqs"])
                for s in op["seqs"]:
                    row = t.row(s)
                    t.ctx[row] += 1
                    t.ctx_bound[row] += 1
                assert op["ok"] and [[k, v] for k, v in counts.items()] == op["counts"]
            except E.PreemptionNeeded as exc:
                assert not op["ok"] and exc.shortfall == op["shortfall"]
        else:
            assert mgr.free_sequence(op["seq"]) == op["freed"]
        got = {str(s): tabs for s, (tabs, _) in t.snapshot().items()}
        assert got == op["tables"]
        assert mgr.free_count == op["free_count"]


@pytest.mark.parametrize("i", range(len(load("decode_cases.json"))))
def test_paged_attention_golden(i):
    """paged_attention + accumulate_decode on the reference's golden inputs."""
    case = load("decode_cases.json")[i]
    st = state_from_snapshot(case["before"], case["num_blocks"], case["block_size"],
                             case["head_dim"], case["layers"], case["heads"])
    st.keys = bf16_round(st.keys)
    st.values = bf16_round(st.values)
    st.metric = st.metric.astype(np.float32).astype(np.float64)
    q = bf16_round(dec(case["query"]))
    rig = DevRig(case["num_blocks"], case["block_size"], case["head_dim"], case["layers"], case["heads"])
    rig.load(st)
    cfg = K.AttentionConfig(case["heads"] * case["r"], case["heads"], case["head_dim"], case["layers"])
    out, rows = K.paged_attention(q, rig.cache, rig.tables, case["seq"], case["layer"], cfg)
    assert isinstance(out, np.ndarray) and all(isinstance(rw, np.ndarray) for rw in rows)  # NumPy in, NumPy out
    ref_out, ref_rows = O.paged_decode(st, q, case["seq"], case["layer"])
    assert np.abs(as_np(out) - ref_out).max() < OUT_ATOL
    for rw, rr in zip(rows, ref_rows):
        assert rw.shape == rr.shape
        assert np.abs(as_np(rw) - rr).max() < ATOL
    mcfg = K.MetricConfig(mode="full", aggregation=case["aggregation"])
    K.accumulate_decode(rig.store, rig.tables, case["seq"], case["layer"], rows, mcfg)
    O.accumulate(st, case["seq"], case["layer"], ref_rows, case["aggregation"])
    got = rig.store.metrics_flat.cpu().numpy()
    assert np.allclose(got, st.metric, rtol=MET_RTOL, atol=1e-6)


CONFIGS = [
    # (b, d, heads, r, max_len, splits)
    (16, 128, 8, 4, 300, 0),
    (16, 128, 2, 4, 2000, 4),
    (16, 128, 2, 8, 1500, 16),
    (16, 64, 4, 4, 700, 2),
    (16, 256, 2, 2, 200, 0),
    (4, 32, 2, 3, 90, 3),
    (2, 16, 4, 1, 50, 0),
    (16, 8, 1, 8, 100, 2),
    # fast path with group sizes off the r in {1,2,4,8} metric kernels:
    # generic metric pass, odd output shares per CTA
    (16, 128, 2, 3, 900, 0),
    (16, 64, 3, 6, 1200, 0),
    (16, 128, 4, 1, 800, 0),
]


@pytest.mark.parametrize("b,d,heads,r,max_len,splits", CONFIGS)
def test_fused_decode_step_matches_oracle(b, d, heads, r, max_len, splits):
    """Fused append + attention + L2 metric over several layers and steps."""
    rng = np.random.default_rng(b * 1000 + d + r)
    layers = 2
    seqs = [3, 1, 7]
    nblocks = 3 * layers * heads * (max_len // b + 4) + 64
    st = random_state(rng, nblocks, b, d, layers, heads, seqs, max_len)
    rig = DevRig(nblocks, b, d, layers, heads)
    rig.load(st)
    cfg = K.AttentionConfig(heads * r, heads, d, layers)
    n_q = heads * r
    for step in range(3):
        # allocation for the step (reference order), then per-layer decode
        want = O.alloc_decode(st, seqs)
        got = rig.manager.allocate_decode_step(seqs)
        assert got == want
        for layer in range(layers):
            q = bf16_round(rng.standard_normal((len(seqs), n_q, d)))
            kn = bf16_round(rng.standard_normal((len(seqs), heads, d)))
            vn = bf16_round(rng.standard_normal((len(seqs), heads, d)))
            dev = rig.cache.device
            out = K.paged_decode(torch.from_numpy(q).to(dev, torch.bfloat16), rig.cache, rig.tables, seqs,
                                 layer, cfg, store=rig.store, metric_mode=2,
                                 k_new=torch.from_numpy(kn).to(dev, torch.bfloat16),
                                 v_new=torch.from_numpy(vn).to(dev, torch.bfloat16),
                                 out_f32=True, splits=splits)
            for i, s in enumerate(seqs):
                ref_out, _ = O.decode_step_layer(st, s, layer, q[i], kn[i], vn[i], "L2")
                err = np.abs(out[i].cpu().numpy() - ref_out).max()
                assert err < OUT_ATOL, err
        from paper_2410_00161_b200 import _lib
        _lib.DeviceContext.get(rig.cache.device).raise_status()
        dst = rig.to_oracle()
        assert_same_ints(dst, st)
        assert np.allclose(dst.metric, st.metric, rtol=MET_RTOL, atol=1e-6)
        for s in seqs:
            for m in range(layers):
                for h in range(heads):
                    f = st.live_slots(s, m, h)
                    assert np.array_equal(dst.keys[f], st.keys[f])
                    assert np.array_equal(dst.values[f], st.values[f])
        # end of step: clear the created-this-step shield (targeted variant)
        rig.store.clear_fresh(rig.tables, seqs)
        O.clear_fresh(st)
        assert np.array_equal(rig.store.fresh_flat.cpu().numpy(), st.fresh)


def test_decode_bf16_output_and_no_metric():
    rng = np.random.default_rng(5)
    b, d, heads, r, layers = 16, 128, 8, 4, 1
    st = random_state(rng, 4096, b, d, layers, heads, [0, 1], 1000)
    rig = DevRig(4096, b, d, layers, heads)
    rig.load(st)
    cfg = K.AttentionConfig(heads * r, heads, d, layers)
    q = bf16_round(rng.standard_normal((2, heads * r, d)))
    out = K.paged_decode(torch.from_numpy(q).to("cuda", torch.bfloat16), rig.cache, rig.tables, [0, 1], 0, cfg)
    for i, s in enumerate([0, 1]):
        ref, _ = O.paged_decode(st, q[i], s, 0)
        assert np.abs(out[i].float().cpu().numpy() - ref).max() < 1e-2
    # metrics untouched without metric_mode
    assert np.array_equal(rig.store.metrics_flat.cpu().numpy(), st.metric.astype(np.float32))


def test_error_paths():
    rig = DevRig(8, 4, 8, 1, 1)
    cfg = K.AttentionConfig(1, 1, 8, 1)
    rig.tables.add_sequence(0)
    rig.manager._take(0, 0, 0)
    with pytest.raises(E.EmptyContextError):
        K.paged_attention(np.zeros((1, 8)), rig.cache, rig.tables, 0, 0, cfg)
    with pytest.raises(E.NumericError):
        K.paged_attention(np.full((1, 8), np.nan), rig.cache, rig.tables, 0, 0, cfg)
    # append beyond the allocated block
    for i in range(4):
        K.append_kv(rig.tables, rig.cache, 0, 0, 0, np.ones(8), np.ones(8))
    with pytest.raises(E.AllocationOrderError):
        K.append_kv(rig.tables, rig.cache, 0, 0, 0, np.ones(8), np.ones(8))
    # pool exhaustion -> PreemptionNeeded with the shortfall, nothing allocated
    mgr = rig.manager
    free = mgr.free_count
    with pytest.raises(E.PreemptionNeeded) as exc:
        mgr.allocate_prefill(1, 4 * (free + 2))
    assert exc.value.shortfall == 2 and mgr.free_count == free and not rig.tables.has_sequence(1)
    with pytest.raises(E.BlockOwnershipError):
        mgr.free_blocks([7])


def test_append_lookup_round_trip():
    rng = np.random.default_rng(7)
    rig = DevRig(256, 4, 8, 3, 2)
    rig.tables.add_sequence(0)
    written = {}
    for layer in range(3):
        for head in range(2):
            n = int(rng.integers(1, 30))
            keys = bf16_round(rng.standard_normal((n, 8)))
            vals = bf16_round(rng.standard_normal((n, 8)))
            for i in range(n):
                if i % 4 == 0:
                    rig.manager._take(0, layer, head)
                h = K.append_kv(rig.tables, rig.cache, 0, layer, head, keys[i], vals[i])
                rig.store.on_append(h, logical=i)
            written[(layer, head)] = (keys, vals)
    for _ in range(200):
        layer, head = int(rng.integers(0, 3)), int(rng.integers(0, 2))
        keys, vals = written[(layer, head)]
        pos = int(rng.integers(0, len(keys)))
        k, v = K.lookup_kv(rig.tables, rig.cache, 0, layer, head, pos)
        assert np.array_equal(k.double().cpu().numpy(), keys[pos])
        assert np.array_equal(v.double().cpu().numpy(), vals[pos])
    assert K.fragmentation(rig.tables) == sum(
        (-(-len(kv[0]) // 4)) * 4 - len(kv[0]) for kv in written.values())


def test_decode_bench_scale_path():
    """The bench's launch configuration: 64 sequences x 8 KV heads (512 pairs)
    with ~1.2-1.6k ragged contexts selects 256-position split-KV items and one
    finish CTA per (sequence, head); a fragmented pool.  Two layers, one
    decode step each, vs the oracle."""
    rng = np.random.default_rng(64)
    b, d, heads, r, layers = 16, 64, 8, 4, 2
    seqs = list(range(64))
    # random_state pre-takes ~30% of the pool to fragment it: size for that
    nblocks = int(len(seqs) * layers * heads * (1700 // b + 2) * 1.6) + 64
    st = random_state(rng, nblocks, b, d, layers, heads, seqs, 1600, min_len=1200)
    rig = DevRig(nblocks, b, d, layers, heads, max_seqs=72, max_blocks=1700 // b + 8)
    rig.load(st)
    cfg = K.AttentionConfig(heads * r, heads, d, layers)
    assert rig.manager.allocate_decode_step(seqs) == O.alloc_decode(st, seqs)
    dev = rig.cache.device
    for layer in range(layers):
        q = bf16_round(rng.standard_normal((len(seqs), heads * r, d)))
        kn = bf16_round(rng.standard_normal((len(seqs), heads, d)))
        vn = bf16_round(rng.standard_normal((len(seqs), heads, d)))
        out = K.paged_decode(torch.from_numpy(q).to(dev, torch.bfloat16), rig.cache, rig.tables, seqs, layer, cfg,
                             store=rig.store, metric_mode=2, k_new=torch.from_numpy(kn).to(dev, torch.bfloat16),
                             v_new=torch.from_numpy(vn).to(dev, torch.bfloat16), out_f32=True).cpu().numpy()
        for i, s in enumerate(seqs):
            ref_out, _ = O.decode_step_layer(st, s, layer, q[i], kn[i], vn[i], "L2")
            assert np.abs(out[i] - ref_out).max() < OUT_ATOL, (layer, s)
    from paper_2410_00161_b200 import _lib
    _lib.DeviceContext.get(dev).raise_status()
    dst = rig.to_oracle()
    assert_same_ints(dst, st)
    assert np.allclose(dst.metric, st.metric, rtol=MET_RTOL, atol=1e-6)


@pytest.mark.parametrize("d", [128, 8])
def test_context_beyond_host_bound_raises(d):
    """A caller that writes tables.ctx directly (the reference tests' idiom)
    past the host bound the launch is sized from: the kernels report
    CacheCorruptionError instead of silently attending a truncated context
    (fast path d = 128: items x score rows; generic path d = 8: chunks)."""
    b, heads, r = 16, 1, 4
    rig = DevRig(128, b, d, 1, heads)
    cfg = K.AttentionConfig(heads * r, heads, d, 1)
    rig.manager.allocate_prefill(0, 64 * b)            # 64 blocks = 1024 slots per head
    rig.tables.set_context_len(0, 0, 0, 100)           # host bound 100
    row = rig.tables.row(0)
    rig.tables.ctx[row, 0, 0] = 900                    # raw write, bound not raised
    q = torch.zeros((1, heads * r, d), dtype=torch.bfloat16, device="cuda")
    K.paged_decode(q, rig.cache, rig.tables, [0], 0, cfg)
    from paper_2410_00161_b200 import _lib
    with pytest.raises(E.CacheCorruptionError):
        _lib.DeviceContext.get(rig.cache.device).raise_status()
    # within the bound it runs
    rig.tables.set_context_len(0, 0, 0, 900)
    K.paged_decode(q, rig.cache, rig.tables, [0], 0, cfg)
    _lib.DeviceContext.get(rig.cache.device).raise_status()


def test_decode_step_raises_bound_once_per_step():
    """paged_decode over every layer of a step raises the row's host context
    bound by one, not by the number of layers (scratch and tables are sized
    from it)."""
    rng = np.random.default_rng(11)
    b, d, heads, r, layers = 16, 64, 2, 2, 4
    st = random_state(rng, 1024, b, d, layers, heads, [0], 100, min_len=50)
    rig = DevRig(1024, b, d, layers, heads)
    rig.load(st)
    cfg = K.AttentionConfig(heads * r, heads, d, layers)
    row = rig.tables.row(0)
    before = rig.tables.ctx_bound[row]
    dev = rig.cache.device
    for _ in range(3):
        rig.manager.allocate_decode_step([0])
        for m in range(layers):
            q = torch.zeros((1, heads * r, d), dtype=torch.bfloat16, device=dev)
            kv = torch.zeros((1, heads, d), dtype=torch.bfloat16, device=dev)
            K.paged_decode(q, rig.cache, rig.tables, [0], m, cfg, store=rig.store, metric_mode=2, k_new=kv,
                           v_new=kv)
    assert rig.tables.ctx_bound[row] == before + 3
    assert int(rig.tables.ctx[row].max()) <= before + 3


def test_layer_chain_equals_stand_alone_launches():
    """A decode step's layers issued as a chain (kvc_decode_args.early_pull 2
    for the first, 1 after: 2-stage ring, a spare CTA slot, early pulls) give
    bit-identical outputs, K/V, tables and metrics to the same layers issued
    stand-alone (early_pull 0: 3-stage ring, no early pull), at d = 128."""
    rng = np.random.default_rng(128)
    b, d, heads, r, layers = 16, 128, 8, 4, 4
    seqs = list(range(16))
    nblocks = int(len(seqs) * layers * heads * (900 // b + 2) * 1.6) + 64
    st = random_state(rng, nblocks, b, d, layers, heads, seqs, 800, min_len=300)
    cfg = K.AttentionConfig(heads * r, heads, d, layers)
    qs = [bf16_round(rng.standard_normal((len(seqs), heads * r, d))) for _ in range(layers)]
    kns = [bf16_round(rng.standard_normal((len(seqs), heads, d))) for _ in range(layers)]
    vns = [bf16_round(rng.standard_normal((len(seqs), heads, d))) for _ in range(layers)]
    results = []
    for chain in (False, True):
        rig = DevRig(nblocks, b, d, layers, heads, max_seqs=24, max_blocks=900 // b + 8)
        rig.load(st)
        rig.manager.allocate_decode_step(seqs)
        dev = rig.cache.device
        rows_t = torch.tensor([rig.tables.row(s) for s in seqs], dtype=torch.int32, device=dev)
        host_rows = [rig.tables.row(s) for s in seqs]
        outs = []
        for layer in range(layers):
            t = lambda x: torch.from_numpy(x).to(dev, torch.bfloat16)
            outs.append(K.paged_decode(t(qs[layer]), rig.cache, rig.tables, seqs, layer, cfg, store=rig.store,
                                       metric_mode=2, k_new=t(kns[layer]), v_new=t(vns[layer]), out_f32=True,
                                       rows_tensor=rows_t, host_rows=host_rows,
                                       early_pull=(1 if layer > 0 else 2) if chain else 0))
        from paper_2410_00161_b200 import _lib
        _lib.DeviceContext.get(dev).raise_status()
        results.append(([o.cpu().numpy() for o in outs], rig.to_oracle()))
    (o0, s0), (o1, s1) = results
    for a, c in zip(o0, o1):
        assert np.array_equal(a, c)
    assert_same_ints(s0, s1)
    assert np.array_equal(s0.metric, s1.metric)
    assert np.array_equal(s0.keys, s1.keys) and np.array_equal(s0.values, s1.values)
