"""DecodeStepGraph (CUDA-graph replay of allocation + every layer + fresh
clear) vs the same steps through paged_decode (GPU).

Integer state (tables, ctx, free list, logical, flags) must match exactly;
outputs and metrics within the decode tolerances (the graph sizes its score
rows for `headroom` more steps, which can change the split-KV partition)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from gpu_rig import DevRig, random_state

pytestmark = pytest.mark.gpu

import paper_2410_00161_b200 as K  # noqa: E402
from paper_2410_00161_b200 import _lib  # noqa: E402


@pytest.mark.parametrize("host", [False, True])
@pytest.mark.parametrize("seqs,max_len,headroom", [([3, 1, 7], 300, 4), ([0, 2, 5, 9], 1200, 64)])
def test_graph_step_equals_eager(seqs, max_len, headroom, host):
    b, d, layers, heads, r = 16, 128, 2, 4, 4
    rng = np.random.default_rng(len(seqs) * 100 + max_len)
    nblocks = 3 * layers * heads * len(seqs) * (max_len // b + 12) + 64
    st = random_state(rng, nblocks, b, d, layers, heads, seqs, max_len)
    rigs = [DevRig(nblocks, b, d, layers, heads, max_seqs=16), DevRig(nblocks, b, d, layers, heads, max_seqs=16)]
    for rig in rigs:
        rig.load(st)
    cfg = K.AttentionConfig(heads * r, heads, d, layers)
    dev = rigs[0].cache.device
    B, n_q = len(seqs), heads * r
    host_io = None
    if host:  # two pinned host sets, used alternately (per-layer upload/download inside the step)
        host_io = [{"q": torch.empty((layers, B, n_q, d), dtype=torch.bfloat16).pin_memory(),
                    "k_new": torch.empty((layers, B, heads, d), dtype=torch.bfloat16).pin_memory(),
                    "v_new": torch.empty((layers, B, heads, d), dtype=torch.bfloat16).pin_memory(),
                    "out": torch.empty((layers, B, n_q, d), dtype=torch.bfloat16).pin_memory()} for _ in range(2)]
    g = K.DecodeStepGraph(rigs[0].cache, rigs[0].tables, rigs[0].manager, rigs[0].store, seqs, cfg,
                          headroom=headroom, host_io=host_io)
    steps = 2 * headroom + 3  # crosses at least one recapture
    for step in range(steps):
        q = torch.randn((layers, B, n_q, d), device=dev).to(torch.bfloat16)
        kn = torch.randn((layers, B, heads, d), device=dev).to(torch.bfloat16)
        vn = torch.randn((layers, B, heads, d), device=dev).to(torch.bfloat16)
        if host:
            h = host_io[step % 2]
            torch.cuda.synchronize()  # the set's previous step has finished with it
            h["q"].copy_(q), h["k_new"].copy_(kn), h["v_new"].copy_(vn)
            g.step(io=step % 2)
            torch.cuda.synchronize()
            out_g = h["out"].to(dev)
        else:
            g.q.copy_(q), g.k_new.copy_(kn), g.v_new.copy_(vn)
            out_g = g.step().clone()
        e = rigs[1]
        e.manager.allocate_decode_step(seqs, sync=False)
        out_e = torch.empty_like(out_g)
        for m in range(layers):
            K.paged_decode(q[m], e.cache, e.tables, seqs, m, cfg, store=e.store, metric_mode=2, k_new=kn[m],
                           v_new=vn[m], fresh=True, out=out_e[m])
        e.store.clear_fresh(e.tables, seqs)
        _lib.DeviceContext.get(dev).raise_status()
        assert (out_g.float() - out_e.float()).abs().max().item() < 2e-2, step
    a, c = rigs[0].to_oracle(), rigs[1].to_oracle()
    assert a.tables == c.tables
    for s in seqs:
        assert np.array_equal(a.ctx[s], c.ctx[s])
    assert np.array_equal(a.free, c.free)
    assert np.array_equal(a.logical, c.logical)
    assert np.array_equal(a.fresh, c.fresh) and np.array_equal(a.protected, c.protected)
    assert np.array_equal(a.keys, c.keys) and np.array_equal(a.values, c.values)
    assert np.allclose(a.metric, c.metric, rtol=1e-3, atol=1e-6)
    assert g.replays == steps - 1
