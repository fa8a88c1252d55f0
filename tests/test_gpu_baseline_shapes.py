"""Parity at the BASELINE.json shapes the bench numbers come from (GPU).

* K2 over all 32 layers x 8 KV heads x 32k prompt tokens (r = 4, d = 128):
  one persistent multi-layer call, the regime where every CTA holds 14-15
  of its 16 TMEM score slots and the slot ring wraps across layers; every
  layer against the oracle's window restatement (metrics.py:68-89).
* K1 through the captured decode step (DecodeStepGraph) at B = 64, H = 8,
  d = 128 with the ragged per-head contexts a real K2 -> K3 -> K4 round
  leaves (Llama-3.1-8B shapes at 8x: C ~ 4k, r = 4; Llama-3.1-70B shapes at
  64x: C ~ 2k, r = 8), over 20 steps so every head opens new blocks:
  allocation (tables, free pool) and ctx for all 64 sequences exactly, and
  outputs, K/V, metrics, logical indices and flags of sampled sequences
  against oracle states extracted from the device before the first step
  (attention.py:92-127, metrics.py:189-211, block_manager.py:74-97).
* KVC-full at L = 4096 and a ragged 4100 (metrics.py:92-109).

Tolerances as in the other GPU tests: outputs 1e-2 absolute (P enters the
P.V product in bf16), metrics 1e-3 / 2e-3 relative, integers exact.
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

RTOL_WIN = 2e-3
OUT_ATOL = 1e-2
MET_RTOL = 1e-3


def _randn(shape, gen, dev="cuda"):
    return torch.randn(shape, generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16)


def test_window_metric_l8b_all_layers_32k():
    """K2 at the bench shape: 32 layers x 8 heads x 32768, one call."""
    layers, H, r, d, L, w = 32, 8, 4, 128, 32768, 8
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2024)
    q = _randn((layers, H * r, w, d), gen)
    k = _randn((layers, H, L, d), gen)
    cfg = K.MetricConfig()
    out = torch.empty((layers, H, L), dtype=torch.float32, device="cuda")
    K.prefill._window_call(q, k, cfg, H, d, torch.device("cuda"), metrics_out=out)
    _lib.DeviceContext.get(out.device).raise_status()
    for layer in range(layers):
        want, _ = O.window_metric(q[layer].double().cpu().numpy(), k[layer].double().cpu().numpy(), H, w,
                                  cfg.pool, "L2")
        got = out[layer].cpu().numpy().astype(np.float64)
        assert np.allclose(got, want, rtol=RTOL_WIN, atol=1e-6 * want.max()), (layer, np.abs(got - want).max())


# ---------------------------------------------------------------------------
# K1 through the decode-step graph at B = 64
# ---------------------------------------------------------------------------


def _meta_state(rig, seqs) -> O.OracleState:
    """Allocator-only oracle state mirroring the device (head_dim 1)."""
    st = O.OracleState(rig.num_blocks, rig.b, 1, rig.layers, rig.heads)
    st.free = rig.manager.free_flag.cpu().numpy().astype(bool)
    snap = rig.tables.snapshot()
    for s in seqs:
        st.tables[s], st.ctx[s] = snap[s][0], snap[s][1].copy()
    return st


def _mini_state(rig, s, spare_per_head) -> O.OracleState:
    """One sequence's heads copied from the device into a compact oracle state
    (its own block numbering, `spare_per_head` free blocks per head)."""
    b, l, H, d = rig.b, rig.layers, rig.heads, rig.d
    tabs, ctx = rig.tables.snapshot()[s]
    used = sum(len(t) for row in tabs for t in row)
    st = O.OracleState(used + l * H * spare_per_head, b, d, l, H)
    ids = np.array([blk for row in tabs for t in row for blk in t], dtype=np.int64)
    dev_slots = torch.from_numpy((ids[:, None] * b + np.arange(b)).reshape(-1)).cuda()
    n = dev_slots.numel()
    st.keys[:n] = rig.cache.keys_flat[dev_slots].double().cpu().numpy()
    st.values[:n] = rig.cache.values_flat[dev_slots].double().cpu().numpy()
    st.metric[:n] = rig.store.metrics_flat[dev_slots].double().cpu().numpy()
    st.logical[:n] = rig.store.logical_flat[dev_slots].cpu().numpy()
    st.protected[:n] = rig.store.protected_flat[dev_slots].cpu().numpy()
    st.fresh[:n] = rig.store.fresh_flat[dev_slots].cpu().numpy()
    st.free[: used] = False
    st.tables[s] = []
    pos = 0
    for m in range(l):
        st.tables[s].append([])
        for h in range(H):
            nb = len(tabs[m][h])
            st.tables[s][m].append(list(range(pos, pos + nb)))
            pos += nb
    st.ctx[s] = ctx.astype(np.int64).copy()
    return st


def _compare_positions(rig, s, mini):
    """Every live position of every head: device slot vs oracle slot."""
    b = rig.b
    tabs, ctx = rig.tables.snapshot()[s]
    assert np.array_equal(ctx, mini.ctx[s])
    dev_f, ora_f = [], []
    for m in range(rig.layers):
        for h in range(rig.heads):
            c = int(ctx[m, h])
            pos = np.arange(c)
            dev_f.append(np.asarray(tabs[m][h], dtype=np.int64)[pos // b] * b + pos % b)
            ora_f.append(mini.live_slots(s, m, h))
    dev_f = torch.from_numpy(np.concatenate(dev_f)).cuda()
    ora_f = np.concatenate(ora_f)
    assert np.array_equal(rig.cache.keys_flat[dev_f].double().cpu().numpy(), mini.keys[ora_f])
    assert np.array_equal(rig.cache.values_flat[dev_f].double().cpu().numpy(), mini.values[ora_f])
    assert np.array_equal(rig.store.logical_flat[dev_f].cpu().numpy(), mini.logical[ora_f])
    assert np.array_equal(rig.store.protected_flat[dev_f].cpu().numpy(), mini.protected[ora_f])
    assert np.array_equal(rig.store.fresh_flat[dev_f].cpu().numpy(), mini.fresh[ora_f])
    got = rig.store.metrics_flat[dev_f].double().cpu().numpy()
    assert np.allclose(got, mini.metric[ora_f], rtol=MET_RTOL, atol=1e-6), np.abs(got - mini.metric[ora_f]).max()


@pytest.mark.parametrize("r,L,rate", [
    (4, 32768, 8),    # Llama-3.1-8B shapes, 32k, 8x: C ~ 4096 per head
    (8, 131072, 64),  # Llama-3.1-70B shapes (GQA 8:1), 128k, 64x: C ~ 2048 per head
])
def test_decode_graph_at_baseline_shape(r, L, rate):
    B, layers, H, d, b = 64, 2, 8, 128, 16
    steps = 20
    keep = int(L / rate)
    nb_keep = layers * H * (keep // b + 4)
    num_blocks = B * (nb_keep + layers * H * 3) + layers * H * (L // b) + 4096
    rig = DevRig(num_blocks, b, d, layers, H, max_seqs=B + 2, max_blocks=L // b + 8)
    cfg = K.AttentionConfig(H * r, H, d, layers)
    mcfg = K.MetricConfig()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(r * 1000 + rate)
    seqs = list(range(B))
    # every sequence through the real pipeline: prompt -> K2 window metric ->
    # K3 schedule -> K4 compaction to the 1/rate budget (ragged per head)
    for s in seqs:
        q = _randn((layers, H * r, 8, d), gen)
        k = _randn((layers, H, L, d), gen)
        v = _randn((layers, H, L, d), gen)
        E = K.budget_to_blocks(keep, layers, H, b, layers * H * (L // b))
        K.prefill_compress_sequence(rig.cache, rig.tables, rig.manager, rig.store, s, q, k, v, mcfg, E, sync=False)
        del q, k, v
    torch.cuda.synchronize()
    _lib.DeviceContext.get(rig.cache.device).raise_status()
    K.compression.refresh_ctx_bounds(rig.tables, seqs)
    ctx0 = rig.tables.ctx[rig.tables.rows_tensor(seqs).long()].cpu().numpy()
    assert ctx0.min() >= b and ctx0.max() > ctx0.min()  # ragged, every head live
    assert abs(ctx0.mean() - keep) < 0.02 * keep

    meta = _meta_state(rig, seqs)
    checked = seqs[::9]  # 0, 9, ..., 63
    minis = {s: _mini_state(rig, s, spare_per_head=3) for s in checked}

    graph = K.DecodeStepGraph(rig.cache, rig.tables, rig.manager, rig.store, seqs, cfg, metric_mode=2,
                              headroom=steps + 8)
    for step in range(steps):
        qs = _randn(tuple(graph.q.shape), gen)
        ks = _randn(tuple(graph.k_new.shape), gen)
        vs = _randn(tuple(graph.v_new.shape), gen)
        graph.q.copy_(qs)
        graph.k_new.copy_(ks)
        graph.v_new.copy_(vs)
        out = graph.step()
        torch.cuda.synchronize()
        _lib.DeviceContext.get(rig.cache.device).raise_status()
        # allocation + ctx for the whole batch, exactly
        O.alloc_decode(meta, seqs)
        for s in seqs:
            meta.ctx[s] += 1
        snap = rig.tables.snapshot()
        for s in seqs:
            assert snap[s][0] == meta.tables[s], (step, s)
            assert np.array_equal(snap[s][1], meta.ctx[s]), (step, s)
        assert np.array_equal(rig.manager.free_flag.cpu().numpy().astype(bool), meta.free)
        # numerics of the sampled sequences
        qh, kh, vh = qs.double().cpu().numpy(), ks.double().cpu().numpy(), vs.double().cpu().numpy()
        oh = out.float().cpu().numpy()
        for s in checked:
            mini = minis[s]
            O.alloc_decode(mini, [s])
            for m in range(layers):
                ref, _ = O.decode_step_layer(mini, s, m, qh[m, s], kh[m, s], vh[m, s], "L2")
                err = np.abs(oh[m, s] - ref).max()
                assert err < OUT_ATOL, (step, s, m, err)
            O.clear_fresh(mini)
    for s in checked:
        _compare_positions(rig, s, minis[s])


# ---------------------------------------------------------------------------
# KVC-full beyond 1024 tokens
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("L", [4096, 4100])
def test_full_metric_long(L):
    H, r, d, v = 2, 4, 128, 10
    rng = np.random.default_rng(L)
    q = bf16_round(rng.standard_normal((H * r, L, d)))
    k = bf16_round(rng.standard_normal((H, L, d)))
    cfg = K.MetricConfig(mode="full", aggregation="L2", excluded=v)
    got, _ = K.full_metrics_qk(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), cfg, H)
    _lib.DeviceContext.get(got.device).raise_status()
    want = O.full_metric(q, k, H, v, "L2")
    g = got.cpu().numpy().astype(np.float64)
    assert np.allclose(g, want, rtol=RTOL_WIN, atol=1e-6 * want.max()), np.abs(g - want).max()
