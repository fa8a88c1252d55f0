"""K2 observation-window metric (tcgen05) + prefill install vs the CPU oracle (GPU).

Inputs are bf16 on both sides; the oracle computes in float64.  Tolerance:
metrics rtol 2e-3 (fp32 accumulation and exp2 in the kernel), protected
masks and logical indices exact.
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

RTOL = 2e-3

CASES = [
    # (H, r, d, L, window, pool, agg)
    (8, 4, 128, 4100, 8, 7, "L2"),
    (2, 4, 128, 1000, 8, 7, "L1"),
    (1, 8, 128, 777, 8, 3, "L2"),
    (4, 2, 64, 300, 16, 7, "L2"),
    (2, 1, 64, 129, 1, 1, "L2"),
    (2, 4, 128, 5, 8, 7, "L2"),
    (1, 4, 64, 1, 8, 7, "L1"),
    (2, 8, 64, 2050, 8, 5, "L1"),
    (1, 2, 256, 400, 8, 7, "L2"),
]


@pytest.mark.parametrize("H,r,d,L,window,pool,agg", CASES)
def test_window_metric_matches_oracle(H, r, d, L, window, pool, agg):
    rng = np.random.default_rng(H * 100 + L)
    w = min(window, L)
    q = bf16_round(rng.standard_normal((H * r, L, d)))
    k = bf16_round(rng.standard_normal((H, L, d)))
    cfg = K.MetricConfig(mode="window", aggregation=agg, window=window, pool=pool)
    got, prot = K.window_metrics_qk(torch.from_numpy(q[:, L - w:]).cuda(), torch.from_numpy(k).cuda(), cfg, H)
    _lib.DeviceContext.get(got.device).raise_status()
    want, wprot = O.window_metric(q[:, L - w:], k, H, window, pool, agg)
    g = got.cpu().numpy().astype(np.float64)
    assert np.allclose(g, want, rtol=RTOL, atol=1e-6 * want.max()), np.abs(g - want).max()
    assert np.array_equal(prot.cpu().numpy(), wprot)


def test_prefill_install_then_compress_exact():
    """prefill_sequence (scatter + K2 + install) then a compression round;
    the schedule must equal the oracle's on the device-computed metrics."""
    rng = np.random.default_rng(42)
    layers, H, r, d, b, L = 2, 4, 4, 128, 16, 1500
    nblocks = layers * H * (L // b + 2) + 16
    rig = DevRig(nblocks, b, d, layers, H, max_seqs=2)
    q = bf16_round(rng.standard_normal((layers, H * r, L, d)))
    k = bf16_round(rng.standard_normal((layers, H, L, d)))
    v = bf16_round(rng.standard_normal((layers, H, L, d)))
    cfg = K.MetricConfig()
    t = lambda x: torch.from_numpy(x).to("cuda", torch.bfloat16)
    K.prefill_sequence(rig.cache, rig.tables, rig.manager, rig.store, 0, t(q[:, :, L - 8:]), t(k), t(v), cfg)
    _lib.DeviceContext.get(rig.cache.device).raise_status()
    st = O.OracleState(nblocks, b, d, layers, H)
    O.prefill(st, 0, q, k, v)
    dst = rig.to_oracle()
    assert dst.tables == st.tables
    assert np.array_equal(dst.ctx[0], st.ctx[0])
    assert np.array_equal(dst.keys, st.keys) and np.array_equal(dst.values, st.values)
    assert np.array_equal(dst.logical, st.logical)
    assert np.array_equal(dst.protected, st.protected)
    assert np.allclose(dst.metric, st.metric, rtol=RTOL, atol=1e-6 * st.metric.max())
    # identical metrics from here on: schedules must agree exactly
    st.metric = dst.metric.copy()
    E = O.budget_to_blocks(L // 8, layers, H, b, st.block_count(0))
    got = K.compress(rig.cache, rig.tables, rig.manager, rig.store, {0: E}).to_dict()
    assert got == O.compress(st, {0: E})


@pytest.mark.parametrize("layers,H,r,d,L", [
    (3, 8, 4, 128, 4100), (4, 2, 4, 64, 9000), (2, 8, 8, 128, 1500),
    (2, 8, 4, 128, 40000),   # > 16 tiles per CTA: each layer streamed twice (recompute mode)
    (2, 8, 8, 128, 20000),   # r*w = 64 columns, > 8 tiles per CTA: recompute mode
])
def test_window_metric_multi_layer(layers, H, r, d, L):
    """One K2 call over several layers (the persistent kernel streams layer
    l+1 while layer l is finished) equals the oracle layer by layer."""
    rng = np.random.default_rng(layers * 1000 + L)
    w = 8
    q = bf16_round(rng.standard_normal((layers, H * r, w, d)))
    k = bf16_round(rng.standard_normal((layers, H, L, d)))
    cfg = K.MetricConfig()
    out = torch.empty((layers, H, L), dtype=torch.float32, device="cuda")
    t = lambda x: torch.from_numpy(x).to("cuda", torch.bfloat16)
    K.prefill._window_call(t(q), t(k), cfg, H, d, torch.device("cuda"), metrics_out=out)
    _lib.DeviceContext.get(out.device).raise_status()
    g = out.cpu().numpy().astype(np.float64)
    for layer in range(layers):
        want, _ = O.window_metric(q[layer], k[layer], H, w, cfg.pool, "L2")
        assert np.allclose(g[layer], want, rtol=RTOL, atol=1e-6 * want.max()), (layer, np.abs(g[layer] - want).max())
