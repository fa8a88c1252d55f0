"""Reference-signature prompt-metric surface vs the REFERENCE's own outputs (GPU).

tests/golden/metric_cases.json holds, for 24 random shapes (d = 4..16,
L = 1..79), the inputs and the outputs the reference itself produced:
gqa_attention (attention.py:62-89) -> window_metrics (metrics.py:68-89) and
full_metrics (metrics.py:92-109).  Here the same calls go through the
facade: kvc_gqa_attention builds the attention tensor, kvc_attn_metrics
reduces it.  Tolerance: fp32 arithmetic against the reference's float64,
rtol 1e-4 + atol 1e-6; protected masks exact.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_io import dec, load

pytestmark = pytest.mark.gpu

import paper_2410_00161_b200 as K  # noqa: E402
from paper_2410_00161_b200 import errors as E  # noqa: E402

CASES = load("metric_cases.json")


@pytest.mark.parametrize("i", range(len(CASES)))
def test_attention_tensor_metrics_match_reference(i):
    c = CASES[i]
    H, r, L, d = c["heads"], c["r"], c["L"], c["d"]
    q, k = dec(c["q"]), dec(c["k"])
    cfg = K.AttentionConfig(H * r, H, d, 1)
    out, attn = K.gqa_attention(q, k, np.zeros_like(k), cfg)
    a = attn.cpu().numpy().astype(np.float64)
    assert np.allclose(a.sum(axis=2), 1.0, atol=1e-5)
    assert np.all(np.triu(a, 1) == 0.0)
    assert np.all(out.cpu().numpy() == 0.0)
    wcfg = K.MetricConfig(mode="window", aggregation=c["aggregation"], window=c["window"], pool=c["pool"])
    wm, prot = K.window_metrics(attn, wcfg, H)
    want = dec(c["window_metrics"])
    assert np.allclose(wm.cpu().numpy(), want, rtol=1e-4, atol=1e-6), np.abs(wm.cpu().numpy() - want).max()
    assert np.array_equal(prot.cpu().numpy().astype(int), np.asarray(c["protected"]))
    fcfg = K.MetricConfig(mode="full", aggregation=c["aggregation"], excluded=c["excluded"])
    fm = K.full_metrics(attn, fcfg, H)
    want = dec(c["full_metrics"])
    assert np.allclose(fm.cpu().numpy(), want, rtol=1e-4, atol=1e-6), np.abs(fm.cpu().numpy() - want).max()
    pm, pp = K.prompt_metrics(attn, fcfg, H)
    assert torch.equal(pm, fm) and not pp.any()


def test_gqa_attention_output_and_numeric_error():
    rng = np.random.default_rng(3)
    H, r, L, d = 2, 3, 40, 16
    q, k, v = (rng.standard_normal(s) for s in ((H * r, L, d), (H, L, d), (H, L, d)))
    out, attn = K.gqa_attention(q, k, v, K.AttentionConfig(H * r, H, d, 1))
    # out = attn @ v per group (float64 check of the fp32 kernel)
    a = attn.cpu().numpy().astype(np.float64)
    want = np.concatenate([a[h * r:(h + 1) * r] @ v[h] for h in range(H)])
    assert np.allclose(out.cpu().numpy(), want, atol=1e-5)
    q[1, 5, 0] = np.nan
    with pytest.raises(E.NumericError):
        K.gqa_attention(q, k, v, K.AttentionConfig(H * r, H, d, 1))
