"""KVC-full metric (csrc/fullmetric.cu on tcgen05) vs the CPU
oracle's restatement of full_metrics (metrics.py:92-109), itself pinned to
the reference by the metric golden cases (GPU).

Inputs are bf16 on both sides; the oracle computes in float64.  Tolerance:
rtol 2e-3 plus atol 1e-6 x max (fp32 accumulation, ex2.approx)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from gpu_rig import DevRig, bf16_round
from oracle import kvc_oracle as O

pytestmark = pytest.mark.gpu

import paper_2410_00161_b200 as K  # noqa: E402
from paper_2410_00161_b200 import _lib  # noqa: E402

CASES = [
    # (H, r, d, L, excluded, agg)
    (2, 4, 128, 300, 10, "L2"),
    (1, 2, 64, 129, 0, "L1"),
    (4, 2, 64, 1000, 10, "L2"),
    (2, 4, 128, 5, 10, "L2"),     # L <= v: every metric is 0
    (1, 8, 128, 513, 3, "L1"),
    (2, 4, 128, 1024, 10, "L2"),
]


@pytest.mark.parametrize("H,r,d,L,v,agg", CASES)
def test_full_metric_matches_oracle(H, r, d, L, v, agg):
    rng = np.random.default_rng(H * 1000 + L + v)
    q = bf16_round(rng.standard_normal((H * r, L, d)))
    k = bf16_round(rng.standard_normal((H, L, d)))
    cfg = K.MetricConfig(mode="full", aggregation=agg, excluded=v)
    got, prot = K.full_metrics_qk(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), cfg, H)
    _lib.DeviceContext.get(got.device).raise_status()
    want = O.full_metric(q, k, H, excluded=v, aggregation=agg)
    g = got.cpu().numpy().astype(np.float64)
    assert np.allclose(g, want, rtol=2e-3, atol=1e-6 * max(want.max(), 1e-30)), np.abs(g - want).max()
    assert not prot.any()


def test_full_prefill_install():
    """prefill_sequence in full mode installs the KVC-full metric per slot
    (logical = position, nothing protected) like the oracle's prefill."""
    rng = np.random.default_rng(3)
    layers, H, r, d, b, L = 2, 2, 4, 64, 16, 400
    nblocks = layers * H * (L // b + 2) + 16
    rig = DevRig(nblocks, b, d, layers, H, max_seqs=2)
    q = bf16_round(rng.standard_normal((layers, H * r, L, d)))
    k = bf16_round(rng.standard_normal((layers, H, L, d)))
    v = bf16_round(rng.standard_normal((layers, H, L, d)))
    cfg = K.MetricConfig(mode="full", excluded=10)
    t = lambda x: torch.from_numpy(x).to("cuda", torch.bfloat16)
    K.prefill_sequence(rig.cache, rig.tables, rig.manager, rig.store, 0, t(q), t(k), t(v), cfg)
    _lib.DeviceContext.get(rig.cache.device).raise_status()
    st = O.OracleState(nblocks, b, d, layers, H)
    O.prefill(st, 0, q, k, v, mode="full", excluded=10)
    dst = rig.to_oracle()
    assert dst.tables == st.tables
    assert np.array_equal(dst.logical, st.logical)
    assert np.array_equal(dst.protected, st.protected) and not dst.protected.any()
    assert np.allclose(dst.metric, st.metric, rtol=2e-3, atol=1e-6 * st.metric.max())
