"""Same-box sanity bound for K1: FlashInfer's paged decode over the very same
bf16 pool, tables and ragged per-head contexts.

FlashInfer pages are shared by all KV heads of a request; KV-Compress gives
every (sequence, KV head) its own block table and length.  The mapping used
here: every (sequence, KV head) is one FlashInfer request with one KV head and
r query heads (GQA group r), pages = that head's blocks, page size 16, NHD
layout [N, 16, 1, d] - a view of our [N, 16, d] pool, no copy.  Both kernels
read the same bytes; attention only (no append, no metric) on both sides.

Contexts: one layer of the bench's ragged per-head lengths
(profiles/ctx_l8b_b64.json, from real prefill -> K2 -> K3 -> K4 rounds).
Prints one JSON line; profiles/r2_flashinfer_compare.json keeps it.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import paper_2410_00161_b200 as K

    dev = torch.device("cuda")
    ctx = json.load(open(os.path.join(ROOT, "profiles", "ctx_l8b_b64.json")))
    B, l, H = ctx["shape"]
    r, d, b = 4, 128, 16
    layers = int(os.environ.get("FI_LAYERS", "4"))  # distinct layers, so no layer's KV is L2-resident
    C = np.array(ctx["ctx_before"], dtype=np.int64).reshape(B, l, H)[:, :layers, :]
    B = int(os.environ.get("FI_BATCH", B))  # smaller batches: the first B sequences
    C = C[:B]
    nblk = (C + b - 1) // b
    N = int(nblk.sum()) + 64
    cache = K.UnifiedKVCache(N, b, d, device=dev)
    tables = K.BlockTables(layers, H, b, max_seqs=B, max_blocks=int(nblk.max()) + 4, device=dev)
    for s in range(B):
        tables.add_sequence(s)
    perm = np.random.default_rng(3).permutation(N - 64).astype(np.int32)  # fragmented placement
    off = 0
    tab = torch.full(tables.tables.shape, -1, dtype=torch.int32)
    for s in range(B):
        for m in range(layers):
            for h in range(H):
                n = int(nblk[s, m, h])
                tab[s, m, h, :n] = torch.from_numpy(perm[off:off + n])
                off += n
    tables.tables.copy_(tab.to(dev))
    tables.nblocks.copy_(torch.from_numpy(nblk.astype(np.int32)).to(dev))
    tables.ctx.copy_(torch.from_numpy(C.astype(np.int32)).to(dev))
    for s in range(B):
        tables.ctx_bound[tables.row(s)] = int(C[s].max())
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    cache.keys_flat.copy_(torch.randn(cache.keys_flat.shape, generator=g, device=dev).to(torch.bfloat16))
    cache.values_flat.copy_(torch.randn(cache.values_flat.shape, generator=g, device=dev).to(torch.bfloat16))
    cfg = K.AttentionConfig(H * r, H, d, layers)
    q = torch.randn((layers, B, H * r, d), generator=g, device=dev).to(torch.bfloat16)
    bytes_layer = [int(2 * C[:, m, :].sum() * d * 2 + nblk[:, m, :].sum() * 4 + 2 * B * H * r * d * 2)
                   for m in range(layers)]
    ev = lambda: torch.cuda.Event(enable_timing=True)

    hold_ms = float(os.environ.get("FI_HOLD_MS", "40"))

    def timeit(fn, reps=20):
        # device time: a spin kernel holds the stream while the host enqueues
        # every timed launch (small batches are otherwise host-launch bound
        # for both libraries: one Python call per layer)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        torch.cuda._sleep(int(hold_ms * 1.9e6))
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    outs = [torch.empty((B, H * r, d), dtype=torch.bfloat16, device=dev) for _ in range(layers)]
    rows = list(range(B))
    rows_t = torch.tensor([tables.row(s) for s in rows], dtype=torch.int32, device=dev)

    def ours():
        for m in range(layers):
            # consecutive layers on one stream, as a decode step issues them
            # (layer m > 0 may pull work early; kvc_decode_args.early_pull)
            K.paged_decode(q[m], cache, tables, rows, m, cfg, metric_mode=0, out=outs[m], rows_tensor=rows_t,
                           host_rows=[tables.row(s) for s in rows], early_pull=1 if m > 0 else 2)

    t_ours = timeit(ours)
    res = {"what": __doc__.split("\n\n")[0].replace("\n", " "), "batch": B, "kv_heads": H, "group": r,
           "head_dim": d, "layers_timed": layers, "mean_ctx": float(C.mean()),
           "bytes_per_layer": float(np.mean(bytes_layer)),
           "ours": {"ms_per_layer": t_ours / layers,
                    "gbs": float(np.sum(bytes_layer)) / (t_ours * 1e-3) / 1e9}}
    try:
        import flashinfer
        ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        wrappers, fi_out = [], []
        kv_k = cache.keys.view(N, b, 1, d)
        kv_v = cache.values.view(N, b, 1, d)
        tc = os.environ.get("FI_TENSOR_CORES", "0") == "1"
        for m in range(layers):
            n = torch.from_numpy(nblk[:, m, :].reshape(-1))
            indptr = torch.zeros(B * H + 1, dtype=torch.int32)
            indptr[1:] = torch.cumsum(n, 0).to(torch.int32)
            idx = torch.cat([tab[s, m, h, :int(nblk[s, m, h])] for s in range(B) for h in range(H)])
            last = torch.from_numpy((C[:, m, :].reshape(-1) - (n.numpy() - 1) * b).astype(np.int32))
            w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD", use_tensor_cores=tc)
            w.plan(indptr.to(dev), idx.to(dev), last.to(dev), r, 1, d, b, q_data_type=torch.bfloat16,
                   kv_data_type=torch.bfloat16)
            wrappers.append(w)
            fi_out.append(torch.empty((B * H, r, d), dtype=torch.bfloat16, device=dev))
        qf = [q[m].view(B * H, r, d) for m in range(layers)]

        def theirs():
            for m in range(layers):
                wrappers[m].run(qf[m], (kv_k, kv_v), out=fi_out[m])

        t_fi = timeit(theirs)
        # same answer (both read the same bf16 KV)
        err = float((fi_out[0].view(B, H * r, d).float() - outs[0].float()).abs().max())
        res["flashinfer"] = {"version": flashinfer.__version__,
                             "api": f"BatchDecodeWithPagedKVCacheWrapper (NHD, use_tensor_cores={tc})",
                             "ms_per_layer": t_fi / layers,
                             "gbs": float(np.sum(bytes_layer)) / (t_fi * 1e-3) / 1e9,
                             "max_abs_diff_vs_ours": err}
        res["ours_speedup"] = t_fi / t_ours
    except Exception as exc:  # noqa: BLE001 - report, do not hide
        res["flashinfer"] = {"unavailable": f"{type(exc).__name__}: {str(exc)[:300]}"}
    line = json.dumps(res)
    print(line)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "flashinfer_compare.json"), "w") as fh:
        fh.write(line + "\n")


if __name__ == "__main__":
    main()
