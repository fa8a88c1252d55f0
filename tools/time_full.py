"""Time the KVC-full metric (f3) for one layer at Llama-8B shapes
(32 query heads, 8 KV heads, d=128) for several prompt lengths.

Useful flops per layer = 2 passes x n_q x L(L+1)/2 x d x 2 (causal half);
exp2 per layer = 2 x n_q x L(L+1)/2 (one per score in each pass)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_00161_b200 as K  # noqa: E402

H, r, d = 8, 4, 128
res = []
for L in (4096, 8192, 32768):
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    q = torch.randn((H * r, L, d), generator=g, device="cuda", dtype=torch.bfloat16)
    k = torch.randn((H, L, d), generator=g, device="cuda", dtype=torch.bfloat16)
    cfg = K.MetricConfig(mode="full", excluded=10)
    out = torch.empty((H, L), dtype=torch.float32, device="cuda")
    for _ in range(2):
        K.prefill._full_call(q, k, cfg, H, torch.device("cuda"), out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        K.prefill._full_call(q, k, cfg, H, torch.device("cuda"), out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pairs = H * r * L * (L + 1) / 2
    res.append({"L": L, "ms_per_layer": ms, "tflops": 2 * pairs * d * 2 / (ms * 1e-3) / 1e12,
                "gexp_per_s": 2 * pairs / (ms * 1e-3) / 1e9, "ms_per_seq_32_layers": ms * 32})
print(json.dumps(res))
