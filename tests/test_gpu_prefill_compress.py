"""Fused prefill + compress (kvc_prefill_compress) vs prefill_sequence +
compress on the device, and vs the CPU oracle (GPU).

The fused path never writes evicted rows, so K/V is compared on live slots
(logical >= 0) only; everything else - tables, ctx, free flags, metric,
logical, protected, fresh, the schedule record - must be identical.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from gpu_rig import DevRig, bf16_round
from oracle import kvc_oracle as O

pytestmark = pytest.mark.gpu

import paper_2410_00161_b200 as K  # noqa: E402
from paper_2410_00161_b200 import _lib  # noqa: E402


def _run(fused, layers, H, r, d, L, rate, seed, pre_seqs=0):
    rng = np.random.default_rng(seed)
    b = 16
    nblocks = (pre_seqs + 1) * layers * H * (L // b + 2) + 64
    rig = DevRig(nblocks, b, d, layers, H, max_seqs=pre_seqs + 2, max_blocks=L // b + 4)
    t = lambda x: torch.from_numpy(x).to("cuda", torch.bfloat16)
    cfg = K.MetricConfig()
    # earlier sequences fragment the pool first (same on both paths)
    for s in range(pre_seqs):
        q0 = bf16_round(rng.standard_normal((layers, H * r, 8, d)))
        k0 = bf16_round(rng.standard_normal((layers, H, L, d)))
        v0 = bf16_round(rng.standard_normal((layers, H, L, d)))
        K.prefill_sequence(rig.cache, rig.tables, rig.manager, rig.store, s, t(q0), t(k0), t(v0), cfg)
        E0 = K.budget_to_blocks(int(L / rate), layers, H, b, rig.tables.sequence_block_count(s))
        K.compress(rig.cache, rig.tables, rig.manager, rig.store, {s: E0})
    sid = pre_seqs
    q = bf16_round(rng.standard_normal((layers, H * r, 8, d)))
    k = bf16_round(rng.standard_normal((layers, H, L, d)))
    v = bf16_round(rng.standard_normal((layers, H, L, d)))
    blocks = layers * H * -(-L // b)
    E = K.budget_to_blocks(int(L / rate), layers, H, b, blocks)
    if fused:
        sched = K.prefill_compress_sequence(rig.cache, rig.tables, rig.manager, rig.store, sid, t(q), t(k), t(v),
                                            cfg, E)
    else:
        K.prefill_sequence(rig.cache, rig.tables, rig.manager, rig.store, sid, t(q), t(k), t(v), cfg)
        sched = K.compress(rig.cache, rig.tables, rig.manager, rig.store, {sid: E})
    _lib.DeviceContext.get(rig.cache.device).raise_status()
    return rig, sched, (q, k, v, E, sid)


@pytest.mark.parametrize("layers,H,r,d,L,rate,pre", [
    (2, 4, 4, 128, 1500, 4.0, 0),     # short heads: warp-per-head compaction
    (2, 2, 4, 128, 9000, 8.0, 1),     # long heads: k_compact16, fragmented pool
    (1, 8, 4, 64, 2048, 16.0, 0),
])
def test_fused_equals_unfused(layers, H, r, d, L, rate, pre):
    a, sa, _ = _run(True, layers, H, r, d, L, rate, seed=7, pre_seqs=pre)
    b_, sb, _ = _run(False, layers, H, r, d, L, rate, seed=7, pre_seqs=pre)
    assert sa.to_dict() == sb.to_dict()
    x, y = a.to_oracle(), b_.to_oracle()
    assert x.tables == y.tables
    for s in x.ctx:
        assert np.array_equal(x.ctx[s], y.ctx[s])
    assert np.array_equal(x.free, y.free)
    assert np.array_equal(x.metric, y.metric)
    assert np.array_equal(x.logical, y.logical)
    assert np.array_equal(x.protected, y.protected) and np.array_equal(x.fresh, y.fresh)
    live = x.logical >= 0
    assert live.any()
    assert np.array_equal(x.keys[live], y.keys[live]) and np.array_equal(x.values[live], y.values[live])


def test_fused_matches_oracle():
    """Fused path vs the oracle's prefill + compress on the same prompt; the
    oracle's f64 metrics are replaced by the device's fp32 ones first, so the
    schedule, tables, logicals and live K/V must agree exactly."""
    rng = np.random.default_rng(11)
    layers, H, r, d, b, L = 2, 4, 4, 128, 16, 1500
    nblocks = layers * H * (L // b + 2) + 16
    rig = DevRig(nblocks, b, d, layers, H, max_seqs=2)
    q = bf16_round(rng.standard_normal((layers, H * r, L, d)))
    k = bf16_round(rng.standard_normal((layers, H, L, d)))
    v = bf16_round(rng.standard_normal((layers, H, L, d)))
    t = lambda x: torch.from_numpy(x).to("cuda", torch.bfloat16)
    st = O.OracleState(nblocks, b, d, layers, H)
    O.prefill(st, 0, q, k, v)
    E = O.budget_to_blocks(L // 4, layers, H, b, st.block_count(0))
    # device metrics of the same prompt (unfused path) stand in for the f64 ones
    ref = DevRig(nblocks, b, d, layers, H, max_seqs=2)
    K.prefill_sequence(ref.cache, ref.tables, ref.manager, ref.store, 0, t(q[:, :, L - 8:]), t(k), t(v), K.MetricConfig())
    st.metric = ref.to_oracle().metric.copy()
    want = O.compress(st, {0: E})
    got = K.prefill_compress_sequence(rig.cache, rig.tables, rig.manager, rig.store, 0, t(q[:, :, L - 8:]), t(k),
                                      t(v), K.MetricConfig(), E)
    _lib.DeviceContext.get(rig.cache.device).raise_status()
    assert got.to_dict() == want
    dst = rig.to_oracle()
    assert dst.tables == st.tables
    assert np.array_equal(dst.ctx[0], st.ctx[0])
    assert np.array_equal(dst.free, st.free)
    assert np.array_equal(dst.logical, st.logical)
    assert np.array_equal(dst.protected, st.protected)
    assert np.array_equal(dst.metric, st.metric)
    live = st.logical >= 0
    assert np.array_equal(dst.keys[live], st.keys[live]) and np.array_equal(dst.values[live], st.values[live])


def test_fused_full_size_equals_unfused():
    """Llama-3.1-8B shapes at full size (32 layers x 8 heads x 32k, d=128, 8x):
    the fused path leaves the same device state as scatter + K2 + compress
    (compared on the device; live K/V rows bit-identical)."""
    layers, H, r, d, b, L = 32, 8, 4, 128, 16, 32768
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    q = torch.randn((layers, H * r, 8, d), generator=g, device=dev).to(torch.bfloat16)
    k = torch.randn((layers, H, L, d), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((layers, H, L, d), generator=g, device=dev).to(torch.bfloat16)
    E = K.budget_to_blocks(L // 8, layers, H, b, layers * H * (L // b))
    rigs = []
    for fused in (True, False):
        nblocks = layers * H * (L // b) + 64
        rig = DevRig(nblocks, b, d, layers, H, max_seqs=2, max_blocks=L // b + 4)
        if fused:
            s = K.prefill_compress_sequence(rig.cache, rig.tables, rig.manager, rig.store, 0, q, k, v,
                                            K.MetricConfig(), E)
        else:
            K.prefill_sequence(rig.cache, rig.tables, rig.manager, rig.store, 0, q, k, v, K.MetricConfig())
            s = K.compress(rig.cache, rig.tables, rig.manager, rig.store, {0: E})
        _lib.DeviceContext.get(dev).raise_status()
        rigs.append((rig, s.to_dict()))
    (a, sa), (b_, sb) = rigs
    assert sa == sb
    assert sa["freed_blocks"] == E
    ta, tb = a.tables, b_.tables
    assert torch.equal(ta.nblocks, tb.nblocks) and torch.equal(ta.ctx, tb.ctx)
    assert torch.equal(ta.tables[0], tb.tables[0])
    assert torch.equal(a.manager.free_flag, b_.manager.free_flag)
    for x, y in ((a.store.metrics_flat, b_.store.metrics_flat), (a.store.logical_flat, b_.store.logical_flat),
                 (a.store.protected_flat, b_.store.protected_flat), (a.store.fresh_flat, b_.store.fresh_flat)):
        assert torch.equal(x, y)
    live = (a.store.logical_flat >= 0).nonzero().flatten()
    assert live.numel() == layers * H * (L // 8)
    assert torch.equal(a.cache.keys_flat[live], b_.cache.keys_flat[live])
    assert torch.equal(a.cache.values_flat[live], b_.cache.values_flat[live])


@pytest.mark.parametrize("layers,H,r,d,L", [(2, 2, 4, 64, 300), (2, 8, 4, 128, 4100), (1, 4, 8, 128, 1024),
                                             (1, 8, 4, 64, 40000)])
def test_prefill_reads_k_once_equals_scatter(layers, H, r, d, L):
    """prefill_sequence's K2 stores the whole blocks' K rows from its staged
    tiles (write_k; the scatter writes V and each head's partial last block):
    the cache and slot state equal the plain K+V scatter followed by K2.  The
    last shape runs K2's recompute mode (more tiles per CTA than TMEM slots),
    where only the first pass stores."""
    b = 16
    g = torch.Generator(device="cuda")
    g.manual_seed(L + d)
    q = torch.randn((layers, H * r, 8, d), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((layers, H, L, d), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((layers, H, L, d), generator=g, device="cuda").to(torch.bfloat16)
    nb = layers * H * (L // b + 2) + 16
    rigs = []
    for fused_k in (True, False):
        rig = DevRig(nb, b, d, layers, H, max_seqs=2, max_blocks=L // b + 4)
        if fused_k:
            K.prefill_sequence(rig.cache, rig.tables, rig.manager, rig.store, 0, q, k, v, K.MetricConfig())
        else:
            rig.manager.allocate_prefill(0, L)
            K.prefill.write_prefill_kv_layers(rig.cache, rig.tables, 0, k, v)
            p = K.cache.pool_struct(cache=rig.cache, tables=rig.tables, store=rig.store)
            K.prefill._window_call(q, k, K.MetricConfig(), H, d, rig.cache.device, pool_p=p,
                                   seq_row=rig.tables.row(0), layer=0)
        torch.cuda.synchronize()
        _lib.DeviceContext.get(rig.cache.device).raise_status()
        rigs.append(rig)
    a, c = rigs
    assert torch.equal(a.cache.keys, c.cache.keys)
    assert torch.equal(a.cache.values, c.cache.values)
    assert torch.equal(a.store.metrics_flat, c.store.metrics_flat)
    assert torch.equal(a.store.logical_flat, c.store.logical_flat)
    assert torch.equal(a.store.protected_flat, c.store.protected_flat)
    assert torch.equal(a.tables.ctx, c.tables.ctx)
