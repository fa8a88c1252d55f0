"""Time K2 (window metric) alone at Llama-8B shapes: 32 layers x 8 KV heads x 32k, one call."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_00161_b200 as K

H, r, d, L = 8, 4, 128, 32768
nl = int(os.environ.get("K2_LAYERS", "32"))
g = torch.Generator(device="cuda"); g.manual_seed(0)
q = torch.randn((nl, H * r, 8, d), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((nl, H, L, d), generator=g, device="cuda").to(torch.bfloat16)
out = torch.empty((nl, H, L), dtype=torch.float32, device="cuda")
cfg = K.MetricConfig()
for _ in range(3):
    K.prefill._window_call(q, k, cfg, H, d, torch.device("cuda"), metrics_out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    K.prefill._window_call(q, k, cfg, H, d, torch.device("cuda"), metrics_out=out)
e1.record(); torch.cuda.synchronize()
per_layer_us = e0.elapsed_time(e1) * 1e3 / (reps * nl)
print(json.dumps({"twopass": os.environ.get("KVC_K2_TWOPASS"), "layers": nl, "us_per_layer": per_layer_us,
                  "ms_per_sequence": per_layer_us * 32 / 1e3,
                  "GBps": H * L * d * 2 / (per_layer_us * 1e-6) / 1e9}))
