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
from gpu_rig import as_np

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
    assert isinstance(attn, np.ndarray) and attn.dtype == np.float64  # NumPy in, NumPy out
    a = as_np(attn)
    assert np.allclose(a.sum(axis=2), 1.0, atol=1e-5)
    assert np.all(np.triu(a, 1) == 0.0)
    assert np.all(as_np(out) == 0.0)
    wcfg = K.MetricConfig(mode="window", aggregation=c["aggregation"], window=c["window"], pool=c["pool"])
    fcfg = K.MetricConfig(mode="full", aggregation=c["aggregation"], excluded=c["excluded"])
    # once on the NumPy attention (NumPy results), once on a device tensor (device results)
    for att in (attn, torch.as_tensor(attn, dtype=torch.float32, device="cuda")):
        wm, prot = K.window_metrics(att, wcfg, H)
        assert torch.is_tensor(wm) == torch.is_tensor(att)
        want = dec(c["window_metrics"])
        assert np.allclose(as_np(wm), want, rtol=1e-4, atol=1e-6), np.abs(as_np(wm) - want).max()
        assert np.array_equal(as_np(prot).astype(int), np.asarray(c["protected"]))
        fm = K.full_metrics(att, fcfg, H)
        want = dec(c["full_metrics"])
        assert np.allclose(as_np(fm), want, rtol=1e-4, atol=1e-6), np.abs(as_np(fm) - want).max()
        pm, pp = K.prompt_metrics(att, fcfg, H)
        assert np.array_equal(as_np(pm), as_np(fm)) and not as_np(pp).any()


def test_gqa_attention_output_and_numeric_error():
    rng = np.random.default_rng(3)
    H, r, L, d = 2, 3, 40, 16
    q, k, v = (rng.standard_normal(s) for s in ((H * r, L, d), (H, L, d), (H, L, d)))
    out, attn = K.gqa_attention(q, k, v, K.AttentionConfig(H * r, H, d, 1))
    # out = attn @ v per group (float64 check of the fp32 kernel)
    a = as_np(attn)
    want = np.concatenate([a[h * r:(h + 1) * r] @ v[h] for h in range(H)])
    assert np.allclose(as_np(out), want, atol=1e-5)
    # device tensors in: device tensors out, same values
    dv = lambda x: torch.as_tensor(x, dtype=torch.float32, device="cuda")
    out_d, attn_d = K.gqa_attention(dv(q), dv(k), dv(v), K.AttentionConfig(H * r, H, d, 1))
    assert out_d.is_cuda and attn_d.is_cuda
    assert np.array_equal(as_np(attn_d).astype(np.float64), a) and np.array_equal(as_np(out_d).astype(np.float64), as_np(out))
    q[1, 5, 0] = np.nan
    with pytest.raises(E.NumericError):
        K.gqa_attention(q, k, v, K.AttentionConfig(H * r, H, d, 1))
