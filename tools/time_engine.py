"""Engine (f1) throughput: a whole serving workload through the device
Engine vs the reference engine (CPU, when /root/reference is present).

    python tools/time_engine.py [--ref]     # --ref: also time pagedkv's engine (build container only)

Workload: toy shapes (2 layers, 4 KV heads, GQA 2:1, d=64, b=16), 32 requests
with 512-1536-token prompts and 64 output tokens, rate 8, prefill-preempt.
Reports decode tokens/s and steps/s over the whole run (prefills, compression
rounds and preemptions included)."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests", "golden"))
import numpy as np  # noqa: E402
from engine_workload import HashTokens  # noqa: E402

LAYERS, NQ, NK, D, B = 2, 8, 4, 64, 16
rng = np.random.default_rng(0)
REQS = [(int(rng.integers(512, 1536)), 64) for _ in range(32)]
NUM_BLOCKS = 2400


def run(mod, eng_mod, **kw):
    cfg = mod.AttentionConfig(NQ, NK, D, LAYERS)
    eng = eng_mod.Engine(cfg, mod.MetricConfig(), eng_mod.POLICY_PRESETS["prefill-preempt"], NUM_BLOCKS, B, rate=8.0,
                         **kw)
    for i, (pl, ot) in enumerate(REQS):
        eng.submit(HashTokens(2000 + i, pl, ot, LAYERS, NQ, NK, D))
    t0 = time.perf_counter()
    recs = eng.run_to_completion()
    if hasattr(eng, "device"):
        import torch
        torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    toks = sum(r.batch_size for r in recs)
    return {"steps": len(recs), "decode_tokens": toks, "seconds": dt, "tok_per_s": toks / dt,
            "compressions": sum(r.compressions for r in recs), "preemptions": sum(r.preemptions for r in recs)}


out = {}
if "--ref" in sys.argv:
    sys.path.insert(0, "/root/reference/pkg/src")
    import pagedkv
    import pagedkv.engine as RE
    out["reference_cpu"] = run(pagedkv, RE)
else:
    import paper_2410_00161_b200 as K
    run(K, K)  # warm-up (kernel attributes, tensor maps, allocator)
    out["device"] = run(K, K)
    out["device_eager_decode"] = run(K, K, decode_graph=False)
print(json.dumps(out))
