"""Benchmark: compressed paged-attention decode on Llama-3.1-8B shapes.

Workload (BASELINE.json configs[1]): 64 sequences x 32k context per GPU,
32 layers, 8 KV heads, GQA 4:1 (32 query heads), head_dim 128, block size
16, bf16 KV, 8x variable-head-rate compression (per-sequence budget of
L/8 tokens per head on average, allocated across heads by the K3 schedule).

How the compressed state is built (synthetic data, random-init shapes):
  * `--prefill-seqs` sequences go through the real pipeline: 32k-token
    prefill (K/V scatter + K2 window metric on tcgen05) -> K3 schedule ->
    K4 compaction.  Those rounds are timed: the eviction-step numbers.
  * the remaining sequences copy those sequences' per-head lengths (the real
    variable-head-rate raggedness) and are allocated directly.
A decode step = K0 block allocation + 32 x K1 (fused append + paged GQA
attention + L2 metric accumulation) + clearing the step's fresh shields.
`value` = tokens/s with all inputs resident in HBM; `e2e` = the same step
through the public API with queries/new KV copied from pinned host memory
and the attention output copied back every step (`DecodeStepGraph(host_io=)`:
per layer, inside the captured step, overlapping the other layers' attention).  KV (>34 GB) is far larger
than L2, so no flush is needed.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "compressed paged-attn decode tok/s + HBM GB/s; eviction-step ms vs CPU ref"
UNIT = "tok/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64, help="sequences per GPU")
    ap.add_argument("--context", type=int, default=32768)
    ap.add_argument("--rate", type=float, default=8.0)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--group", type=int, default=4)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--prefill-seqs", type=int, default=3, help="real prefill+compress rounds (first = warm-up)")
    ap.add_argument("--splits", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--metric-mode", type=int, default=2, help="decode metric: 2 L2 (reference default), 1 L1, 0 off")
    ap.add_argument("--no-metric-overlap", action="store_true",
                    help="graph step: accumulate the metric in the finish kernel instead of a side branch")
    ap.add_argument("--no-fragmented", action="store_true", help="skip the random-placement decode measurement")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the decode step layer by layer instead of replaying its CUDA graph")
    ap.add_argument("--save-ctx", action="store_true",
                    help="write the decode's per-head starting contexts to profiles/ctx_<preset>_b<B>.json "
                         "(the reference arm decodes the same ragged lengths)")
    ap.add_argument("--preset", default="l8b", choices=sorted(PRESETS),
                    help="BASELINE.json config the shape flags default to (explicit flags override)")
    args = ap.parse_args()
    given = {a.split("=")[0].lstrip("-").replace("-", "_") for a in sys.argv[1:] if a.startswith("--")}
    for k, v in PRESETS[args.preset]["shape"].items():
        if k not in given:
            setattr(args, k, v)
    return args


# BASELINE.json configs as shape presets (configs[1] is the default bench line)
PRESETS = {
    "toy": {"workload": "toy single-layer cache (BASELINE configs[0]): 4 KV heads, d=64, 2 seqs x 1k, 4x",
            "shape": dict(layers=1, kv_heads=4, group=4, head_dim=64, context=1024, rate=4.0, batch=2)},
    "l8b": {"workload": "llama-3.1-8b-shapes decode, 32k ctx, 8x variable-head-rate compression",
            "shape": dict(layers=32, kv_heads=8, group=4, head_dim=128, context=32768, rate=8.0, batch=64)},
    "m7b": {"workload": "mistral-7b-instruct-v0.2 shapes, 32k synthetic prompts, observation-window metric, 16x",
            "shape": dict(layers=32, kv_heads=8, group=4, head_dim=128, context=32768, rate=16.0, batch=64)},
    "l70b": {"workload": "llama-3.1-70b shapes (80 layers, 8 KV heads, GQA 8:1), 128k ctx, 64x, sequences sharded",
             "shape": dict(layers=80, kv_heads=8, group=8, head_dim=128, context=131072, rate=64.0, batch=64)},
}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------


class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._proc = None

    def __enter__(self):
        # one nvidia-smi process sampling every 50 ms for the whole timed region
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self._proc is None:
            return
        time.sleep(0.1)
        self._proc.terminate()
        try:
            out, _ = self._proc.communicate(timeout=5)
        except Exception:
            self._proc.kill()
            out = ""
        for line in (out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:6]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def k1_traffic():
    """DRAM bytes of one K1 layer launch (stream + finish + metric kernels)
    from the newest committed ncu --set full capture (profiles/r*_ncu.json)
    and that file's name, or (None, None)."""
    for name in ("r2_ncu.json", "r1_ncu.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as fh:
                d = json.load(fh)
            return float(sum(r["dram_read_B"] + r["dram_write_B"] for r in d["k1"])), name
        except Exception:
            continue
    return None, None


def build(args, dev, rank):
    import torch
    import paper_2410_00161_b200 as K
    from paper_2410_00161_b200 import _lib

    l, H, r, d, b, L = args.layers, args.kv_heads, args.group, args.head_dim, 16, args.context
    B = args.batch
    n_q = H * r
    keep_tokens = int(L / args.rate)
    hp = l * H
    per_seq_blocks = -(-keep_tokens * hp // b)
    nb_prefill = hp * (-(-L // b))
    growth = hp * (-(-(args.steps + args.warmup + 8) // b) + 2)
    # B running sequences (at least the prefill_seqs compressed ones) + one uncompressed prompt
    num_blocks = int(max(B, args.prefill_seqs) * (per_seq_blocks * 1.25 + growth) + nb_prefill + 4096)
    max_blocks = -(-L // b) + 8
    cache = K.UnifiedKVCache(num_blocks, b, d, device=dev)
    tables = K.BlockTables(l, H, b, max_seqs=max(B, args.prefill_seqs) + 2, max_blocks=max_blocks, device=dev)
    manager = K.BlockManager(num_blocks, tables)
    store = K.MetricsStore(num_blocks, b, device=dev)
    cfg = K.AttentionConfig(n_q, H, d, l)
    mcfg = K.MetricConfig()
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    return dict(K=K, _lib=_lib, torch=torch, cache=cache, tables=tables, manager=manager, store=store, cfg=cfg,
                mcfg=mcfg, gen=gen, l=l, H=H, r=r, d=d, b=b, L=L, B=B, n_q=n_q, keep_tokens=keep_tokens,
                num_blocks=num_blocks)


# spin-kernel length that keeps the stream busy while the host enqueues a
# timed eviction round (~2 ms at the B200's 1965 MHz SM clock)
HOLD_CYCLES = 4_000_000


def eviction_rounds(S, args):
    """Real prefill -> K2 -> K3/K4 for the first sequences; returns timings."""
    torch, K = S["torch"], S["K"]
    cache, tables, manager, store = S["cache"], S["tables"], S["manager"], S["store"]
    l, H, d, L, b = S["l"], S["H"], S["d"], S["L"], S["b"]
    dev = cache.device
    ev = lambda: torch.cuda.Event(enable_timing=True)
    out = {"k2_ms": [], "k34_ms": [], "scatter_ms": [], "freed": [], "moves": [], "evicted": []}
    for s in range(args.prefill_seqs):
        manager.allocate_prefill(s, L)
        q = torch.randn((l, S["n_q"], 8, d), generator=S["gen"], device=dev, dtype=torch.bfloat16)
        k = torch.randn((l, H, L, d), generator=S["gen"], device=dev, dtype=torch.bfloat16)
        v = torch.randn((l, H, L, d), generator=S["gen"], device=dev, dtype=torch.bfloat16)
        e0, e1, e2 = ev(), ev(), ev()
        torch.cuda.synchronize()
        e0.record()
        # the unfused prompt path as prefill_sequence runs it: V (+ each
        # head's partial last K block) scattered, then K2, which stores the
        # whole blocks' K rows from the tiles it streams
        K.prefill.write_prefill_kv_layers(cache, tables, s, k, v, v_only=True)
        e1.record()
        p = K.cache.pool_struct(cache=cache, tables=tables, store=store)
        if not K.prefill._window_call(q, k, S["mcfg"], H, d, dev, pool_p=p, seq_row=tables.row(s), layer=0,
                                      write_k=True):
            sys.exit("bench.py: K2 cannot store the prompt K rows at this shape")
        e2.record()
        # the plain K+V prompt write, timed alone (it rewrites the same rows):
        # what the fused on-prefill step is compared against
        e3, e4 = ev(), ev()
        K.prefill.write_prefill_kv_layers(cache, tables, s, k, v)
        e3.record()
        # the eviction step's metric: K2 alone (recomputes and reinstalls the
        # same metrics, no K write)
        K.prefill._window_call(q, k, S["mcfg"], H, d, dev, pool_p=p, seq_row=tables.row(s), layer=0)
        e4.record()
        torch.cuda.synchronize()
        sc_t = e0.elapsed_time(e1)
        k2_t = e3.elapsed_time(e4)
        out.setdefault("k2_write_k_ms", []).append(e1.elapsed_time(e2))
        out.setdefault("full_scatter_ms", []).append(e2.elapsed_time(e3))
        del k, v
        S["_lib"].DeviceContext.get(dev).raise_status()
        E = K.budget_to_blocks(S["keep_tokens"], l, H, b, tables.sequence_block_count(s))
        e0, e1, e2 = ev(), ev(), ev()
        torch.cuda.synchronize()
        # hold the stream (~2 ms spin kernel) while the host prepares and
        # enqueues the round, so the events time the device work alone (host
        # enqueue is reported separately; an engine overlaps it with decode)
        torch.cuda._sleep(HOLD_CYCLES)
        t_h = time.perf_counter()
        plan = K.compress(cache, tables, manager, store, {s: E}, sync=False, events=(e0, e1))
        out.setdefault("host_enqueue_ms", []).append((time.perf_counter() - t_h) * 1e3)
        # the round's only cross-GPU traffic: all-gather of every rank's
        # (freed, evicted, moves, free) counters, stream-ordered under NCCL
        out["rank_counts"] = K.gather_round_counts(plan.totals)
        e2.record()
        torch.cuda.synchronize()
        S["_lib"].DeviceContext.get(dev).raise_status()
        tot = plan.totals.tolist()
        K.compression.refresh_ctx_bounds(tables, [s])
        out["k2_ms"].append(k2_t)
        out["scatter_ms"].append(sc_t)
        out["k34_ms"].append(e0.elapsed_time(e2))
        out.setdefault("k34_kernels_ms", []).append(e0.elapsed_time(e1))
        out["freed"].append(tot[0])
        out["evicted"].append(tot[1])
        out["moves"].append(tot[2])
    # the same prefill + compress fused (kvc_prefill_compress): evicted rows are
    # never written and survivors never moved; a spare table row, freed after
    out["fused_ms"] = []
    for i in range(args.prefill_seqs):
        sid = 1_000_000 + i
        q = torch.randn((l, S["n_q"], 8, d), generator=S["gen"], device=dev, dtype=torch.bfloat16)
        k = torch.randn((l, H, L, d), generator=S["gen"], device=dev, dtype=torch.bfloat16)
        v = torch.randn((l, H, L, d), generator=S["gen"], device=dev, dtype=torch.bfloat16)
        E = K.budget_to_blocks(S["keep_tokens"], l, H, b, l * H * -(-L // b))
        e0, e1 = ev(), ev()
        torch.cuda.synchronize()
        torch.cuda._sleep(HOLD_CYCLES)
        K.prefill_compress_sequence(cache, tables, manager, store, sid, q, k, v, S["mcfg"], E, sync=False,
                                    events=(e0, e1))
        torch.cuda.synchronize()
        S["_lib"].DeviceContext.get(dev).raise_status()
        out["fused_ms"].append(e0.elapsed_time(e1))
        del k, v
        manager.free_sequence(sid, store=store)
    return out


def populate(S, args):
    """Remaining sequences: copy the compressed sequences' per-head lengths."""
    torch = S["torch"]
    tables, manager = S["tables"], S["manager"]
    P = args.prefill_seqs
    templates = [(tables.nblocks[tables.row(s)].clone(), tables.ctx[tables.row(s)].clone()) for s in range(P)]
    for s in range(P, S["B"]):
        nb, ctx = templates[s % P]
        tables.add_sequence(s)
        manager._alloc_heads(s, nb.flatten().cpu())
        row = tables.row(s)
        tables.ctx[row] = ctx
        tables.ctx_bound[row] = int(ctx.max())
    # per-slot metadata (metric, logical, protected) copied block by block
    # from the template head, so the copies are valid compress() inputs
    store, b = S["store"], S["b"]
    mt, lg, pr = store.metrics.view(-1), store.logical.view(-1), store.protected_u8.view(-1)
    off = torch.arange(b, device=tables.tables.device, dtype=torch.int64)
    jj = torch.arange(tables.max_blocks, device=tables.tables.device)
    for s in range(P, S["B"]):
        t = s % P
        nb = tables.nblocks[tables.row(t)]
        live = (jj[None, None, :] < nb[..., None].long())
        src = (tables.tables[tables.row(t)].long()[live][:, None] * b + off).reshape(-1)
        dst = (tables.tables[tables.row(s)].long()[live][:, None] * b + off).reshape(-1)
        mt[dst], lg[dst], pr[dst] = mt[src], lg[src], pr[src]
    # fill every pool block with unit-normal bf16 (K/V of the copied heads)
    cache = S["cache"]
    kf, vf = cache.keys.view(-1), cache.values.view(-1)
    step = 1 << 28
    for t in (kf, vf):
        for o in range(0, t.numel(), step):
            t[o: o + step].normal_(generator=S["gen"])
    torch.cuda.synchronize()


def decode_bytes(S, ctx_host):
    """Algorithmic bytes of one K1 launch per layer given per-head C (before append)."""
    d, b = S["d"], S["b"]
    C = ctx_host + 1  # attended keys incl. the appended one
    kv = 2 * C * d * 2
    table = -(-C // b) * 4
    metric = 2 * C * 4
    qo = S["B"] * 2 * S["n_q"] * d * 2
    new_kv = S["B"] * S["H"] * 2 * d * 2
    per_layer = (kv + table + metric).reshape(S["B"], S["l"], S["H"]).sum(axis=(0, 2))
    return per_layer + qo + new_kv  # [l]


def decode_bench(S, args, e2e=False):
    torch, K = S["torch"], S["K"]
    cache, tables, manager, store, cfg = S["cache"], S["tables"], S["manager"], S["store"], S["cfg"]
    dev = cache.device
    B, l, H, n_q, d = S["B"], S["l"], S["H"], S["n_q"], S["d"]
    seqs = list(range(B))
    rows = [tables.row(s) for s in seqs]
    rows_t = torch.tensor(rows, dtype=torch.int32, device=dev)
    steps, warm = args.steps, args.warmup
    # inputs: one set per step (resident in HBM for `value`; pinned host for e2e)
    n_sets = 2
    gen = S["gen"]
    q = [torch.randn((l, B, n_q, d), generator=gen, device=dev).to(torch.bfloat16) for _ in range(n_sets)]
    kn = [torch.randn((l, B, H, d), generator=gen, device=dev).to(torch.bfloat16) for _ in range(n_sets)]
    vn = [torch.randn((l, B, H, d), generator=gen, device=dev).to(torch.bfloat16) for _ in range(n_sets)]
    out = torch.empty((l, B, n_q, d), dtype=torch.bfloat16, device=dev)
    if e2e:
        hq = [x.cpu().pin_memory() for x in q]
        hk = [x.cpu().pin_memory() for x in kn]
        hv = [x.cpu().pin_memory() for x in vn]
        hout = torch.empty(out.shape, dtype=torch.bfloat16).pin_memory()
        houts = [hout] + [torch.empty(out.shape, dtype=torch.bfloat16).pin_memory() for _ in range(n_sets - 1)]
        dq, dk, dv = torch.empty_like(q[0]), torch.empty_like(kn[0]), torch.empty_like(vn[0])
    ctx_host = tables.ctx[rows_t.long()].cpu().numpy().astype(np.int64).reshape(-1)  # [B*l*H]
    layer_events = []
    # default: the whole step (allocation + every layer + fresh clear) replayed
    # as one CUDA graph; its static input buffers are written every step
    graph = None
    if not args.no_graph:
        # e2e: the graph uploads each layer's Q/K/V from the pinned host set and
        # downloads its output inside the step, overlapped with the other layers
        host_io = ([{"q": hq[i], "k_new": hk[i], "v_new": hv[i], "out": houts[i]} for i in range(n_sets)]
                   if e2e else None)
        graph = K.DecodeStepGraph(cache, tables, manager, store, seqs, cfg, metric_mode=args.metric_mode,
                                  headroom=max(64, args.steps + args.warmup + 8),
                                  metric_overlap=not args.no_metric_overlap, host_io=host_io)

    def one_step(i, timed):
        sel = i % n_sets
        if graph is not None:
            if e2e:
                graph.step(io=sel)
                return
            graph.q.copy_(q[sel])
            graph.k_new.copy_(kn[sel])
            graph.v_new.copy_(vn[sel])
            graph.step()
            return
        manager.allocate_decode_step(seqs, sync=False)
        if e2e:
            dq.copy_(hq[sel], non_blocking=True)
            dk.copy_(hk[sel], non_blocking=True)
            dv.copy_(hv[sel], non_blocking=True)
            qq, kk, vv = dq, dk, dv
        else:
            qq, kk, vv = q[sel], kn[sel], vn[sel]
        for m in range(l):
            if timed and not e2e:
                a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
            K.paged_decode(qq[m], cache, tables, None, m, cfg, store=store, metric_mode=args.metric_mode, k_new=kk[m],
                           v_new=vv[m], fresh=True, out=out[m], rows_tensor=rows_t, host_rows=rows,
                           splits=args.splits)
            if timed and not e2e:
                z.record()
                layer_events.append((a, z))
        _clear_fresh_rows(S, rows_t)
        if e2e:
            hout.copy_(out, non_blocking=True)

    for i in range(warm):
        one_step(i, False)
    torch.cuda.synchronize()
    S["_lib"].DeviceContext.get(dev).raise_status()
    ctx_before = tables.ctx[rows_t.long()].cpu().numpy().astype(np.int64).reshape(-1)
    if S.get("dist"):
        S["dist"].barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cvd = [x for x in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if x.strip()]
    cur = torch.cuda.current_device()
    clocks = Clocks(int(cvd[cur]) if cur < len(cvd) and cvd[cur].strip().isdigit() else cur)
    with clocks:
        torch.cuda.synchronize()
        t0.record()
        for i in range(steps):
            one_step(warm + i, True)
        t1.record()
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    S["_lib"].DeviceContext.get(dev).raise_status()
    res = {"ms": ms, "clocks": clocks.summary(), "ctx_before": ctx_before}
    if not e2e:
        bytes_steps = np.stack([decode_bytes(S, ctx_before + i) for i in range(steps)])  # [steps, l]
        res["k1_bytes_mean"] = float(bytes_steps.mean())
        res["bytes_per_step"] = float(bytes_steps.sum(axis=1).mean())
        if graph is None:
            durs = np.array([a.elapsed_time(z) for a, z in layer_events]).reshape(steps, l)
            res["k1_ms_mean"] = float(durs.mean())
            res["k1_gbs"] = float(bytes_steps.sum() / (durs.sum() * 1e-3) / 1e9)
            res["k1_timing"] = "CUDA events around each layer's launches (stream, finish) on the launching stream"
        else:
            # inside the replay a layer cannot be bracketed by events: charge K1
            # the whole step (input copies, allocation and fresh clear included)
            res["k1_ms_mean"] = float(ms / steps / l)
            res["k1_gbs"] = float(bytes_steps.sum() / (ms * 1e-3) / 1e9)
            res["k1_timing"] = ("CUDA-graph replay: decode step time / layers, CUDA events around the timed "
                                "steps (input copies, K0 allocation and fresh clear charged to K1)")
        # K0 (decode demand, tile scan, tile take, bind) + per layer K1 (stream, finish[, metric on the
        # graph's side branch]) + fresh clear
        per_layer = 3 if (graph is not None and graph.metric_overlap) else 2
        res["launches_per_step"] = 4 + per_layer * l + 1
    else:
        res["h2d"] = int(sum(x.numel() * 2 for x in (hq[0], hk[0], hv[0])))
        res["d2h"] = int(hout.numel() * 2)
    return res


def fragment_placement(S, seed=7):
    """Randomly permute the physical blocks behind every running sequence's
    tables (post-compaction fragmentation vs sequential
    placement).  Only the table -> block mapping changes; block contents are
    synthetic, so decode work is identical."""
    torch = S["torch"]
    tables = S["tables"]
    rows = torch.tensor([tables.row(s) for s in range(S["B"])], device=tables.tables.device).long()
    tab = tables.tables[rows]                                   # [B, l, H, maxB]
    nb = tables.nblocks[rows].long()
    live = torch.arange(tab.shape[-1], device=tab.device)[None, None, None, :] < nb[..., None]
    ids = tab[live]
    g = torch.Generator(device=ids.device)
    g.manual_seed(seed)
    tab[live] = ids[torch.randperm(ids.numel(), generator=g, device=ids.device)]
    tables.tables[rows] = tab
    torch.cuda.synchronize()


def decode_compression_rounds(S, args, rounds=2, gap_steps=8):
    """The engine's every-step policy (engine.py:89-93, 275-280, 360-378):
    one compress() over the whole running batch, budgets from
    budget_to_blocks(prompt_len / rate), metric from decode accumulation.
    `gap_steps` decode steps between rounds give every head new tokens.
    Returns per-round device ms of K3+K4 and the blocks each freed."""
    torch, K = S["torch"], S["K"]
    cache, tables, manager, store, cfg = S["cache"], S["tables"], S["manager"], S["store"], S["cfg"]
    dev = cache.device
    B, l, H, n_q, d, b = S["B"], S["l"], S["H"], S["n_q"], S["d"], S["b"]
    seqs = list(range(B))
    rows = [tables.row(s) for s in seqs]
    rows_t = torch.tensor(rows, dtype=torch.int32, device=dev)
    q = torch.randn((B, n_q, d), generator=S["gen"], device=dev).to(torch.bfloat16)
    kv = torch.randn((B, H, d), generator=S["gen"], device=dev).to(torch.bfloat16)
    out = {"ms": [], "freed": [], "sequences": B}
    for _ in range(rounds):
        for _ in range(gap_steps):
            manager.allocate_decode_step(seqs, sync=False)
            for m in range(l):
                K.paged_decode(q, cache, tables, None, m, cfg, store=store, metric_mode=2, k_new=kv, v_new=kv,
                               fresh=True, rows_tensor=rows_t, host_rows=rows)
            _clear_fresh_rows(S, rows_t)
        nb = tables.nblocks[rows_t.long()].reshape(B, -1).sum(dim=1).tolist()
        budgets = {s: K.budget_to_blocks(S["keep_tokens"], l, H, b, int(nb[i])) for i, s in enumerate(seqs)}
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize()
        torch.cuda._sleep(HOLD_CYCLES)  # device time only (see eviction_rounds)
        plan = K.compress(cache, tables, manager, store, budgets, sync=False, events=(e0, e1))
        K.gather_round_counts(plan.totals)
        e2.record()
        torch.cuda.synchronize()
        S["_lib"].DeviceContext.get(dev).raise_status()
        K.compression.refresh_ctx_bounds(tables, seqs)
        out["ms"].append(e0.elapsed_time(e2))
        out["freed"].append(int(plan.totals.tolist()[0]))
    return out


def _clear_fresh_rows(S, rows_t):
    from paper_2410_00161_b200 import _lib
    import ctypes
    p = S["K"].cache.pool_struct(tables=S["tables"], store=S["store"])
    _lib.check(_lib.lib().kvc_clear_fresh(ctypes.byref(p), rows_t.data_ptr(), rows_t.numel(),
                                          _lib.stream_ptr(S["cache"].device)), "clear_fresh")


# ---------------------------------------------------------------------------
# CPU baselines (the oracle port, bounded samples)
# ---------------------------------------------------------------------------


def cpu_decode_sample(ctx_heads, d, r, H, seconds, seed=0):
    """Oracle decode of one (sequence, layer) with the given per-head C at d;
    returns seconds per (sequence, layer)."""
    from oracle import kvc_oracle as O

    rng = np.random.default_rng(seed)
    b = 16
    total = sum(-(-int(c + 1) // b) for c in ctx_heads) + 8
    st = O.OracleState(total, b, d, 1, H)
    st.tables[0] = [[[] for _ in range(H)]]
    st.ctx[0] = np.zeros((1, H), dtype=np.int64)
    perm = rng.permutation(total)
    pos = 0
    for h, c in enumerate(ctx_heads):
        nb = -(-int(c + 1) // b)
        st.tables[0][0][h] = [int(x) for x in perm[pos: pos + nb]]
        st.free[perm[pos: pos + nb]] = False
        pos += nb
        st.ctx[0][0, h] = int(c)
    st.keys[:] = rng.standard_normal(st.keys.shape)
    st.values[:] = rng.standard_normal(st.values.shape)
    q = rng.standard_normal((H * r, d))
    kn = rng.standard_normal((H, d))
    t0 = time.perf_counter()
    n = 0
    while True:
        O.decode_step_layer(st, 0, 0, q, kn, kn, "L2")
        n += 1
        # undo the append so the sample stays the same size
        st.ctx[0][0] -= 1
        if time.perf_counter() - t0 > seconds:
            break
    return (time.perf_counter() - t0) / n


def cpu_evict_sample(ctx_heads_layer, L, H, layers_sample, rate, seed=0):
    """Oracle schedule+compaction (head_dim 1) of one sequence slice of
    `layers_sample` layers at L tokens; returns seconds for that slice."""
    from oracle import kvc_oracle as O

    rng = np.random.default_rng(seed)
    b = 16
    st = O.OracleState(layers_sample * H * (L // b) + 8, b, 1, layers_sample, H)
    O.alloc_prefill(st, 0, L)
    for m in range(layers_sample):
        for h in range(H):
            st.ctx[0][m, h] = L
            f = st.live_slots(0, m, h)
            st.metric[f] = O.pool_max(rng.random((1, L)) ** 3, 7)[0]
            st.logical[f] = np.arange(L)
            st.protected[f[-8:]] = True
    E = O.budget_to_blocks(int(L / rate), layers_sample, H, b, st.block_count(0))
    t0 = time.perf_counter()
    O.compress(st, {0: E})
    return time.perf_counter() - t0


def cpu_window_sample(L, H, r, d, seed=0):
    from oracle import kvc_oracle as O

    rng = np.random.default_rng(seed)
    q = rng.standard_normal((H * r, 8, d))
    k = rng.standard_normal((H, L, d))
    t0 = time.perf_counter()
    O.window_metric(q, k, H)
    return time.perf_counter() - t0


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------


def config_dict(args, world, shared=False):
    return {"workload": PRESETS[args.preset]["workload"], "preset": args.preset,
            "batch_per_gpu": args.batch, "global_batch": args.batch * world, "context": args.context,
            "layers": args.layers, "kv_heads": args.kv_heads, "query_heads": args.kv_heads * args.group,
            "head_dim": args.head_dim, "block_size": 16, "compression": f"{args.rate:g}x",
            "metric": "window w=8 p=7 L2 at prefill, L2 decode accumulation",
            "parallelism": f"seq-shard x{world}" + (" (ranks sharing one GPU: code-path check, not a measurement)"
                                                      if shared else ""),
            "l2": "KV working set (>34 GB) >> 126 MB L2; no flush needed"}


# ---------------------------------------------------------------------------
# --impl reference: the reference's CPU path (oracle port) on the host cores
# ---------------------------------------------------------------------------


def ctx_fixture_path(args):
    return os.path.join(ROOT, "profiles", f"ctx_{args.preset}_b{args.batch}.json")


def load_ctx_fixture(args):
    """Per-(sequence, layer, head) contexts the GPU arm decodes from (its
    ctx_before, saved by `bench.py --save-ctx`), or None."""
    try:
        with open(ctx_fixture_path(args)) as fh:
            d = json.load(fh)
        a = np.asarray(d["ctx_before"], dtype=np.int64)
        if list(d["shape"]) == [args.batch, args.layers, args.kv_heads] and d["context"] == args.context \
                and d["rate"] == args.rate:
            return a.reshape(args.batch, args.layers, args.kv_heads)
    except Exception:
        pass
    return None


_REF = {}


def _ref_worker_init(H, r, d, max_ctx, seed):
    """A worker's oracle pool: random f64 K/V for 2 units of H heads at the
    largest context (each unit is placed at random blocks of it)."""
    from oracle import kvc_oracle as O

    b = 16
    nb = -(-(max_ctx + 1) // b)
    st = O.OracleState(2 * H * nb + 8, b, d, 1, H)
    rng = np.random.default_rng(seed + os.getpid())
    st.keys[:] = rng.standard_normal(st.keys.shape)
    st.values[:] = rng.standard_normal(st.values.shape)
    st.tables[0] = [[[] for _ in range(H)]]
    st.ctx[0] = np.zeros((1, H), dtype=np.int64)
    _REF.update(O=O, st=st, rng=rng, b=b, r=r)


def _ref_units(units):
    """The reference decode of (seq, layer) units, each = per-head contexts:
    append the step's K/V to every head, attend in table order, fold the L2
    mass into the metrics (engine.py:426-444: append_kv, paged_attention,
    accumulate_decode), then undo the append so every step has the same size."""
    O, st, rng, b = _REF["O"], _REF["st"], _REF["rng"], _REF["b"]
    H, d = st.num_kv_heads, st.head_dim
    r = _REF["r"]
    perm = rng.permutation(st.num_blocks)
    for ctx_heads in units:
        pos = 0
        for h, c in enumerate(ctx_heads):
            nb = -(-(int(c) + 1) // b)
            st.tables[0][0][h] = perm[pos: pos + nb].tolist()
            pos += nb
            st.ctx[0][0, h] = int(c)
        q = rng.standard_normal((H * r, d))
        kn = rng.standard_normal((H, d))
        O.decode_step_layer(st, 0, 0, q, kn, kn, "L2")
        st.ctx[0][0] -= 1
        perm = np.roll(perm, pos)
    return len(units)


def run_reference(args, world):
    """--impl reference: full decode steps of the reference algorithm (the
    oracle port of attention.py:92-127 + metrics.py:189-211, float64 NumPy),
    B sequences x l layers of (sequence, layer) units per step, on every
    host core (one process per core, one BLAS thread each), over the same
    ragged per-head contexts the GPU arm decodes (profiles/ctx_*.json, saved
    from the GPU arm).  At N > 1 a step is one rank's share (B sequences)
    and the job time is that x N (a bounded sample)."""
    import multiprocessing as mp
    import platform

    cores = os.cpu_count() or 1
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"  # one BLAS thread per worker process: no oversubscription
    L, H, r, d, l, B = args.context, args.kv_heads, args.group, args.head_dim, args.layers, args.batch
    ctx = load_ctx_fixture(args)
    ragged = ctx is not None
    if ctx is None:
        ctx = np.full((B, l, H), int(L / args.rate), dtype=np.int64)
    units = [ctx[s, m].tolist() for s in range(B) for m in range(l)]
    n_chunks = min(len(units), cores * 4)
    chunks = [units[i::n_chunks] for i in range(n_chunks)]
    cpu_model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            cpu_model = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), cpu_model)
    except Exception:
        pass
    t_steps = []
    with mp.get_context("spawn").Pool(cores, initializer=_ref_worker_init,
                                      initargs=(H, r, d, int(ctx.max()) + 1, 17)) as pool:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            done = sum(pool.map(_ref_units, chunks, chunksize=1))
            t_steps.append(time.perf_counter() - t0)
            assert done == len(units)
    step_s = float(np.mean(t_steps[args.warmup:])) * world
    value = B * world / step_s
    sample = (f"full decode steps: {B} sequences x {l} layers = {len(units)} (seq, layer) units of oracle "
              f"decode_step_layer (append + paged attention + L2 accumulate, f64) per step, {H} heads, d={d}, "
              + (f"ragged per-head C from the GPU arm's compressed state (mean {ctx.mean():.0f}, "
                 f"{os.path.basename(ctx_fixture_path(args))})" if ragged else f"uniform C={int(L / args.rate)}")
              + f"; {cores} worker processes x 1 BLAS thread on '{cpu_model}'"
              + (f"; N={world}: one rank's share per step, job time x{world}" if world > 1 else ""))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                             "cpu_model": cpu_model, "step_s": t_steps[args.warmup:]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------


def relaunch(args):
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) on
    this node and exit with their status."""
    import socket

    import torch

    shared = os.environ.get("KVC_BENCH_SHARE_GPU") == "1"
    have = torch.cuda.device_count()
    if have < args.gpus and not shared:
        sys.exit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    world = int(world_env or "1")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:  # rank 0 alone times the CPU path; the other ranks exit 0
            run_reference(args, world if world_env else args.gpus)
        return
    if world_env is None and args.gpus > 1:
        relaunch(args)
        return
    if world != args.gpus:
        sys.exit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={world}")
    import torch

    # ranks sharing one GPU (KVC_BENCH_SHARE_GPU=1, gloo): exercises the
    # multi-rank code path on a 1-GPU box; its numbers are not measurements
    shared = os.environ.get("KVC_BENCH_SHARE_GPU") == "1"
    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        if not shared and torch.cuda.device_count() < world:
            sys.exit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} CUDA device(s) visible")
        # NCCL's init log (rank / device / transport lines) goes to stderr so the
        # JSON line stays the last line of stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(0 if shared else local)
        dist_mod.init_process_group("gloo" if shared else "nccl", device_id=None if shared else
                                    torch.device("cuda", local))
        dist = dist_mod
    dev = torch.device("cuda", torch.cuda.current_device())
    S = build(args, dev, rank)
    S["dist"] = dist
    ev = eviction_rounds(S, args)
    populate(S, args)
    dec = decode_bench(S, args)
    if os.environ.get("KVC_BENCH_DECODE_ONLY"):  # experiments: decode timing only
        print("DECODE", {k: v for k, v in dec.items() if not hasattr(v, "shape")}, flush=True)
        return
    if args.save_ctx and rank == 0:
        with open(ctx_fixture_path(args), "w") as fh:
            json.dump({"shape": [args.batch, args.layers, args.kv_heads], "context": args.context, "rate": args.rate,
                       "what": "per-(sequence, layer, head) context C the GPU arm's timed decode starts from "
                               "(3 real prefill->K2->K3->K4 rounds, copied round-robin to the batch)",
                       "ctx_before": dec["ctx_before"].tolist()}, fh)
    e2e = None if args.no_e2e else decode_bench(S, args, e2e=True)
    dcr = decode_compression_rounds(S, args)
    # last: the same decode with every block of the batch at a random place in
    # the pool (metadata no longer needed; the step is otherwise identical)
    frag = None
    if not args.no_fragmented:
        fragment_placement(S)
        fsteps = max(3, min(args.steps, 5))
        fargs = argparse.Namespace(**{**vars(args), "steps": fsteps})
        frag = decode_bench(S, fargs)
        frag["steps"] = fsteps
    timed = slice(1, None) if len(ev["k2_ms"]) > 1 else slice(None)
    mine = {"ms": dec["ms"], "ms_e2e": e2e["ms"] if e2e else None, "frag_ms": frag["ms"] if frag else None,
            "k2": float(np.mean(ev["k2_ms"][timed])), "k34": float(np.mean(ev["k34_ms"][timed])),
            "k34_kernels": float(np.mean(ev["k34_kernels_ms"][timed])),
            "k34_host": float(np.mean(ev["host_enqueue_ms"][timed])),
            "scatter": float(np.mean(ev["scatter_ms"][timed])),
            "full_scatter": float(np.mean(ev["full_scatter_ms"][timed])),
            "k2_write_k": float(np.mean(ev["k2_write_k_ms"][timed])),
            "fused": float(np.mean(ev["fused_ms"][timed])) if ev["fused_ms"] else None,
            "dcr": dcr["ms"][-1], "clocks": dec["clocks"]}
    if dist is not None:  # every rank's numbers to every rank; times are the max over ranks
        allr = [None] * world
        dist.all_gather_object(allr, mine)
    else:
        allr = [mine]
    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return
    tmax = lambda k: max(x[k] for x in allr) if allr[0][k] is not None else None
    rank_counts = ev["rank_counts"].cpu().tolist() if torch.is_tensor(ev["rank_counts"]) else ev["rank_counts"]
    B, steps = args.batch, args.steps
    ms, ms_e2e = tmax("ms"), tmax("ms_e2e")
    value = B * world * steps / (ms * 1e-3)
    peak, peak_kind = peaks()
    step_ms = ms / steps
    k2, k34, k34k, scat, fused = tmax("k2"), tmax("k34"), tmax("k34_kernels"), tmax("scatter"), tmax("fused")
    evict = {
        "per_sequence_ms": {"k2_window_metric": k2, "k3k4_schedule_compact": k34,
                            "k3k4_kernels_only": k34k, "total": k2 + k34, "v_scatter_not_counted": scat, "k2_with_k_write": tmax("k2_write_k"),
                            "k3k4_host_enqueue": tmax("k34_host"),
                            "what": "device time (CUDA events; the stream is held by a spin kernel while the host "
                                    "prepares and enqueues, so host time is not in the device figures and is "
                                    "reported as k3k4_host_enqueue); k3k4 includes the per-round NCCL all-gather "
                                    "of (freed, evicted, moves, free) counters (world > 1); max over ranks"},
        "freed_blocks": ev["freed"], "moves": ev["moves"], "evicted_kvs": ev["evicted"],
        "rank_counts_last_round": rank_counts,
        "rounds_ms": {"k2": ev["k2_ms"], "k3k4": ev["k34_ms"], "first_round_is_warmup": len(ev["k2_ms"]) > 1},
        "prefill_side_per_sequence_ms": {
            "what": "prompt K/V into the cache + window metric + compress to the budget, per new sequence",
            "unfused_scatter_k2_k3k4": scat + tmax("k2_write_k") + k34,
            "unfused_what": "V scatter (+ partial last K block) + K2 (window metric; stores the whole blocks' K rows "
                            "from the tiles it streams) + K3/K4", "fused_prefill_compress": fused,
            "fused_rounds_ms": ev["fused_ms"]},
        "ratio_to_decode_step": {
            "raw_with_k2": (k2 + k34) / step_ms, "raw_without_k2": k34 / step_ms,
            "amortised_500_tokens_with_k2": (k2 + k34) * B / 500 / step_ms},
        "decode_round": {
            "what": f"every-step policy: one compress() over all {B} running sequences "
                    f"(K3+K4, decode-accumulated L2 metric), {8} decode steps after the previous round",
            "ms": tmax("dcr"), "freed_blocks": dcr["freed"], "ratio_to_decode_step": tmax("dcr") / step_ms},
    }
    if fused is not None:
        # on-prefill policy: the metric -> schedule -> compact step fused into the
        # prompt write, minus the plain prompt write it replaces (can be < 0)
        full_scat = tmax("full_scatter")
        evict["fused_marginal_over_prompt_write"] = {
            "ms_per_sequence": fused - full_scat, "ratio_to_decode_step": (fused - full_scat) / step_ms,
            "plain_prompt_write_ms": full_scat,
            "what": "prefill_compress_sequence minus the plain K+V prompt write (write_prefill_kv_layers) of the "
                    "same prompt"}
    frag_line = None
    if frag is not None:
        fsteps = frag["steps"]
        frag_line = {"value": B * world * fsteps / (tmax("frag_ms") * 1e-3), "unit": UNIT,
                     "ms_per_step": tmax("frag_ms") / fsteps, "steps": fsteps,
                     "what": "same decode step with the batch's blocks randomly permuted over the pool "
                             "(fragmented placement; the default line is the allocator's contiguous placement)"}
    # K1 bytes per launch are this rank's; with equal shards every rank moves the same
    k1_gbs = dec["bytes_per_step"] / (step_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (unit-normal Q/K/V, random-init shapes; no checkpoints)",
        "config": config_dict(args, world, shared),
        "per_rank_ms_per_step": [x["ms"] / steps for x in allr],
        "hbm_gbs_decode_step": k1_gbs,
        "roofline": {"bound": "hbm",
                     "kernel": "K1 per layer: k_decode_stream + k_decode_finish (+ k_decode_metric, graph side branch)",
                     "achieved": dec["k1_gbs"] if world == 1 else k1_gbs, "peak": peak, "unit": "GB/s",
                     "frac": (dec["k1_gbs"] if world == 1 else k1_gbs) / peak,
                     "peak_source": peak_kind, "traffic": k1_traffic()[0],
                     "traffic_source": f"profiles/{k1_traffic()[1]}: dram bytes of one K1 layer launch from a "
                                       "committed ncu --set full capture (not measured in this run)",
                     "bytes_per_launch": dec["k1_bytes_mean"], "launch_ms": dec["k1_ms_mean"],
                     "timing": dec["k1_timing"] + ("; per GPU, slowest rank" if world > 1 else "")},
        "eviction_step": evict,
        "fragmented_placement": frag_line,
        "clocks": dec["clocks"],
        "clocks_per_rank": [x["clocks"] for x in allr] if world > 1 else None,
        "gpu_launches": dec["launches_per_step"] * steps,
    }
    if e2e:
        line["e2e"] = {"value": B * world * steps / (ms_e2e * 1e-3), "unit": UNIT,
                       "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"]}
    if not args.no_cpu and world == 1:  # the CPU baseline is an N = 1 figure (rank 0)
        from threadpoolctl import threadpool_limits

        ctx = dec["ctx_before"].reshape(B, args.layers, args.kv_heads)
        with threadpool_limits(limits=1):  # the reference is single-threaded Python/numpy
            t_sl = cpu_decode_sample(ctx[0, 0].tolist(), args.head_dim, args.group, args.kv_heads,
                                     args.cpu_seconds / 2)
            t_ev = cpu_evict_sample(None, args.context, args.kv_heads, 2, args.rate)
            t_w = cpu_window_sample(args.context, args.kv_heads, args.group, args.head_dim)
        line["cpu_baseline"] = {
            "value": 1.0 / (args.layers * t_sl), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": (f"oracle decode_step_layer of one (seq, layer): {args.kv_heads} heads, C={ctx[0, 0].tolist()}, "
                       f"d={args.head_dim}, looped ~{args.cpu_seconds / 2:.0f}s; tok/s = 1/(layers x t); "
                       f"eviction: compress of 2 layers x {args.kv_heads} heads x {args.context} at head_dim 1 "
                       f"(x{args.layers // 2} to a full sequence); window metric of 1 layer (x{args.layers})"),
            "eviction_step_ms_per_sequence": t_ev * 1e3 * args.layers / 2 + t_w * 1e3 * args.layers,
            "schedule_compact_ms_per_sequence": t_ev * 1e3 * args.layers / 2,
            "window_metric_ms_per_sequence": t_w * 1e3 * args.layers,
        }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
