"""Time the prefill K/V scatter alone at Llama-8B shapes (32 layers x 8 heads x 32k, d=128)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_00161_b200 as K

l, H, d, b, L = 32, 8, 128, 16, 32768
nb = l * H * (L // b) * 2 + 4096
dev = torch.device("cuda")
cache = K.UnifiedKVCache(nb, b, d, device=dev)
tables = K.BlockTables(l, H, b, max_seqs=4, max_blocks=L // b + 8, device=dev)
mgr = K.BlockManager(nb, tables)
g = torch.Generator(device=dev); g.manual_seed(0)
k = torch.randn((l, H, L, d), generator=g, device=dev).to(torch.bfloat16)
v = torch.randn((l, H, L, d), generator=g, device=dev).to(torch.bfloat16)
res = []
for s in range(3):
    mgr.allocate_prefill(s, L)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    K.prefill.write_prefill_kv_layers(cache, tables, s, k, v)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    res.append({"ms": ms, "GBps": 4 * k.numel() * 2 / ms / 1e6})
    mgr.free_sequence(s)
print(json.dumps(res))
