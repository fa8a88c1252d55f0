"""Small-shape workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) over every libkvc kernel family: K0 allocator, K1 decode (eager and
the CUDA-graph step with the early pull between layers), K2 window metric
(persistent tcgen05 kernel), KVC-full, K3/K4 compress (per-head block path and
the warp path of decode rounds), the fused prefill+compress and the prompt
scatter.  Run from the repo root:

    compute-sanitizer --tool racecheck python tools/sanitize.py

Results are checked against the oracle by the smoke part (test harness use)."""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import paper_2410_00161_b200 as K
    from paper_2410_00161_b200 import _lib
    from gpu_rig import DevRig, random_state
    from smoke_impl import run_smoke

    run_smoke()  # K1 eager, K3/K4 compress, K2 (persistent), KVC-full
    ctx = _lib.DeviceContext.get(torch.device("cuda", 0))

    # K0 + K1 CUDA-graph step: 2 layers (layer 1 early-pulls behind layer 0's kernel B)
    b, d, layers, heads, r = 16, 128, 2, 4, 4
    seqs = [0, 1, 2]
    rng = np.random.default_rng(7)
    nblocks = 3 * layers * heads * len(seqs) * (300 // b + 12) + 64
    st = random_state(rng, nblocks, b, d, layers, heads, seqs, 300)
    rig = DevRig(nblocks, b, d, layers, heads, max_seqs=8)
    rig.load(st)
    cfg = K.AttentionConfig(heads * r, heads, d, layers)
    g = K.DecodeStepGraph(rig.cache, rig.tables, rig.manager, rig.store, seqs, cfg, headroom=4)
    for _ in range(3):
        g.q.normal_(), g.k_new.normal_(), g.v_new.normal_()
        g.step()
    torch.cuda.synchronize()
    ctx.raise_status()
    # decode-round compress (warp-per-head compaction for short heads)
    E = {s: max(1, int(rig.tables.sequence_block_count(s)) // 4) for s in seqs}
    K.compress(rig.cache, rig.tables, rig.manager, rig.store, E)
    ctx.raise_status()

    # fused prefill + compress and the unfused prompt path: a short prompt
    # (warp-per-head compaction) and a long one (> 8192 slots per head: K3's
    # last-level bounds, k_compact16 and the concurrent K/V copy kernel)
    for L in (700, 9000):
        prompt_rounds(K, DevRig, ctx, L)
    print("sanitize workload done")


def prompt_rounds(K, DevRig, ctx, L):
    b = 16
    H2, r2, d2, l2 = 2, 4, 128, 2
    qf = torch.randn((l2, H2 * r2, 8, d2), device="cuda").to(torch.bfloat16)
    kf = torch.randn((l2, H2, L, d2), device="cuda").to(torch.bfloat16)
    vf = torch.randn((l2, H2, L, d2), device="cuda").to(torch.bfloat16)
    nb = l2 * H2 * (L // b + 2) * 2 + 16
    for fused in (True, False):
        rig2 = DevRig(nb, b, d2, l2, H2, max_seqs=2, max_blocks=L // b + 4)
        if fused:
            K.prefill_compress_sequence(rig2.cache, rig2.tables, rig2.manager, rig2.store, 0, qf, kf, vf,
                                        K.MetricConfig(), L // 16)
        else:
            K.prefill_sequence(rig2.cache, rig2.tables, rig2.manager, rig2.store, 0, qf, kf, vf, K.MetricConfig())
            K.compress(rig2.cache, rig2.tables, rig2.manager, rig2.store, {0: L // 16})
        torch.cuda.synchronize()
        ctx.raise_status()


if __name__ == "__main__":
    main()
