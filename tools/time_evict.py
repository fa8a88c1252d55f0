"""Time one Llama-8B-shaped eviction round (K2 + K3/K4) per sequence, 3 rounds."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_00161_b200 as K
from paper_2410_00161_b200 import _lib

l, H, r, d, b, L = 32, 8, 4, 128, 16, 32768
nb = l * H * (L // b) + 4096
dev = torch.device("cuda")
cache = K.UnifiedKVCache(nb, b, d, device=dev)
tables = K.BlockTables(l, H, b, max_seqs=4, max_blocks=L // b + 8, device=dev)
mgr = K.BlockManager(nb, tables)
store = K.MetricsStore(nb, b, device=dev)
g = torch.Generator(device=dev); g.manual_seed(0)
q = torch.randn((l, H * r, 8, d), generator=g, device=dev).to(torch.bfloat16)
k = torch.randn((l, H, L, d), generator=g, device=dev).to(torch.bfloat16)
v = torch.randn((l, H, L, d), generator=g, device=dev).to(torch.bfloat16)
ev = lambda: torch.cuda.Event(enable_timing=True)
res = []
for rnd in range(4):
    K.prefill_sequence(cache, tables, mgr, store, rnd, q, k, v, K.MetricConfig())
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    p = K.cache.pool_struct(cache=cache, tables=tables, store=store)
    e0.record()
    K.prefill._window_call(q, k, K.MetricConfig(), H, d, dev, pool_p=p, seq_row=tables.row(rnd), layer=0)
    e1.record()
    torch.cuda.synchronize()
    k2 = e0.elapsed_time(e1)
    E = K.budget_to_blocks(L // 8, l, H, b, tables.sequence_block_count(rnd))
    e4, e5 = ev(), ev()
    torch.cuda._sleep(4_000_000)  # hold the stream (~2 ms) so the events time device work, not host enqueue
    e4.record()
    K.compression.schedule_evictions(tables, store, {rnd: E}, manager=mgr)  # K3 alone (no state change)
    e5.record()
    torch.cuda.synchronize()
    e2, e3 = ev(), ev()
    torch.cuda._sleep(4_000_000)
    t0 = time.perf_counter()
    plan = K.compress(cache, tables, mgr, store, {rnd: E}, sync=False, events=(e2, e3))
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    _lib.DeviceContext.get(dev).raise_status()
    res.append({"round": rnd, "k2_ms": k2, "k3_ms": e4.elapsed_time(e5), "k34_ms": e2.elapsed_time(e3), "host_enqueue_ms": (t1 - t0) * 1e3,
                "wall_ms": (t2 - t0) * 1e3, "freed": int(plan.totals[0])})
    mgr.free_sequence(rnd, store=store)
# fused prefill + compress (K2 + K3 + K4 on metadata + survivor placement)
for rnd in range(4, 7):
    e0, e1 = ev(), ev()
    torch.cuda.synchronize()
    torch.cuda._sleep(4_000_000)
    K.prefill_compress_sequence(cache, tables, mgr, store, rnd, q, k, v, K.MetricConfig(),
                                K.budget_to_blocks(L // 8, l, H, b, l * H * (L // b)), sync=False, events=(e0, e1))
    torch.cuda.synchronize()
    _lib.DeviceContext.get(dev).raise_status()
    res.append({"round": rnd, "fused_prefill_compress_ms": e0.elapsed_time(e1)})
    mgr.free_sequence(rnd, store=store)
print(json.dumps(res))
