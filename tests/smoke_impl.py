"""__graft_entry__.smoke(): one small decode step on cuda:0 checked against
the CPU oracle (the oracle is only the checker)."""

from __future__ import annotations

import numpy as np
import torch


def run_smoke():
    from gpu_rig import DevRig, bf16_round, random_state
    from oracle import kvc_oracle as O
    import paper_2410_00161_b200 as K
    from paper_2410_00161_b200 import _lib

    assert torch.cuda.is_available(), "smoke needs cuda:0"
    rng = np.random.default_rng(0)
    b, d, heads, r, layers = 16, 128, 4, 4, 1
    seqs = [0, 1]
    st = random_state(rng, 2048, b, d, layers, heads, seqs, 400)
    rig = DevRig(2048, b, d, layers, heads)
    rig.load(st)
    cfg = K.AttentionConfig(heads * r, heads, d, layers)
    assert rig.manager.allocate_decode_step(seqs) == O.alloc_decode(st, seqs)
    q = bf16_round(rng.standard_normal((2, heads * r, d)))
    kn = bf16_round(rng.standard_normal((2, heads, d)))
    vn = bf16_round(rng.standard_normal((2, heads, d)))
    t = lambda x: torch.from_numpy(x).to("cuda", torch.bfloat16)
    out = K.paged_decode(t(q), rig.cache, rig.tables, seqs, 0, cfg, store=rig.store, metric_mode=2,
                         k_new=t(kn), v_new=t(vn), out_f32=True)
    _lib.DeviceContext.get(rig.cache.device).raise_status()
    for i, s in enumerate(seqs):
        ref, _ = O.decode_step_layer(st, s, 0, q[i], kn[i], vn[i], "L2")
        err = float(np.abs(out[i].cpu().numpy() - ref).max())
        assert err < 1e-2, err  # bf16 P in the P.V MMA
    dst = rig.to_oracle()
    assert np.allclose(dst.metric, st.metric, rtol=1e-3, atol=1e-6)
    # one compression round on the device metrics: schedule must be bit-exact
    st.metric = dst.metric.copy()
    rig.store.clear_fresh(rig.tables, seqs)
    O.clear_fresh(st)
    budgets = {s: O.budget_to_blocks(100, layers, heads, b, st.block_count(s)) for s in seqs}
    got = K.compress(rig.cache, rig.tables, rig.manager, rig.store, budgets).to_dict()
    want = O.compress(st, budgets)
    assert got == want, "compress schedule differs from the oracle"
    # prefill: K/V scatter + K2 window metric (tcgen05, persistent) installed per slot
    L, H2, r2, d2 = 300, 2, 4, 64
    qf = bf16_round(rng.standard_normal((1, H2 * r2, L, d2)))
    kf = bf16_round(rng.standard_normal((1, H2, L, d2)))
    vf = bf16_round(rng.standard_normal((1, H2, L, d2)))
    nb = H2 * (L // b + 2) + 8
    rig2 = DevRig(nb, b, d2, 1, H2, max_seqs=2)
    K.prefill_sequence(rig2.cache, rig2.tables, rig2.manager, rig2.store, 0, t(qf[:, :, L - 8:]), t(kf), t(vf),
                       K.MetricConfig())
    _lib.DeviceContext.get(rig2.cache.device).raise_status()
    st2 = O.OracleState(nb, b, d2, 1, H2)
    O.prefill(st2, 0, qf, kf, vf)
    got2 = rig2.to_oracle()
    assert np.allclose(got2.metric, st2.metric, rtol=2e-3, atol=1e-6 * st2.metric.max()), "window metric"
    # KVC-full metric (tcgen05 row statistics + column sums)
    full, _ = K.full_metrics_qk(t(qf[0]), t(kf[0]), K.MetricConfig(mode="full"), H2)
    want_full = O.full_metric(qf[0], kf[0], H2, excluded=10, aggregation="L2")
    assert np.allclose(full.cpu().numpy(), want_full, rtol=2e-3, atol=1e-6 * want_full.max()), "full metric"
    print("smoke: decode + compress + window/full metric parity ok")
