"""Regenerate profiles/r1_summary.md from the committed evidence files.

    python profiles/make_summary.py
"""
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
J = lambda f: json.load(open(os.path.join(HERE, f)))
b, ref, n, nf, fm, eng = (J("r1_bench.json"), J("r1_bench_reference.json"), J("r1_ncu.json"), J("r1_ncu_full.json"),
                          J("r1_full_metric.json"), J("r1_engine.json"))
peak = json.load(open(os.path.join(HERE, "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(HERE, "..", "MEASURED_PEAKS.json")) else b["roofline"]["peak"]


def row(r):
    t = r["duration_us"]
    tr = r["dram_read_B"] + r["dram_write_B"]
    tc = r["tcgen05_pipe_pct"] if r["tcgen05_pipe_pct"] not in ("0", "n/a") else "-"
    return (f"| `{r['kernel']}` | {t:.1f} | {r['dram_read_B'] / 1e6:.1f} | {r['dram_write_B'] / 1e6:.1f} | "
            f"{tr / t / 1e3:.0f} | {r['dram_pct_of_peak']:.1f}% | {tc} |")


e, r = b["eviction_step"], b["roofline"]
p, ps, dr, fr = e["per_sequence_ms"], e["prefill_side_per_sequence_ms"], e["decode_round"], b["fragmented_placement"]
mg = e.get("fused_marginal_over_prompt_write")
cfg = subprocess.run(["python", os.path.join(HERE, "..", "tools", "summarize_configs.py")], capture_output=True,
                     text=True).stdout
k1tr = sum(x["dram_read_B"] + x["dram_write_B"] for x in n["k1"])
f32 = [x for x in fm if x["L"] == 32768][0]
L = ["# Round 1 — measurements on B200 (one GPU)\n",
     "All numbers come from `gpurun` calls on one B200: 148 SMs, 1965 MHz max SM clock. The default line's",
     f"clock samples: median {b['clocks']['sm_mhz']:.0f} MHz under load, throttle reasons "
     f"{', '.join(b['clocks']['reasons']) or 'none'} (no hw/thermal slowdown).",
     "The roofline denominator is the HBM copy bandwidth the driver measured,",
     f"{peak} GB/s (`MEASURED_PEAKS.json`). A read-only stream reaches more on this part: 6.8 TB/s with",
     "LDG.128 and 7.3 TB/s with TMA (`tools/microbench/readbw.cu`, table below).",
     "Regenerate with `python profiles/make_summary.py`.\n",
     "## bench.py default line (Llama-3.1-8B shapes, B=64 × 32k per GPU, 8x, 32 layers)\n",
     "Source: `profiles/r1_bench.json`. The reference arm is in `profiles/r1_bench_reference.json`.\n",
     "| quantity | value |", "|---|---|",
     f"| decode throughput | **{b['value']:.0f} tok/s** ({b['ms_per_step']:.2f} ms per step; the step is one CUDA-graph replay) |",
     f"| K1 achieved bandwidth | {r['achieved']:.0f} GB/s = **{r['frac'] * 100:.1f}%** of the measured HBM copy rate. "
     f"Basis: {r['bytes_per_launch'] / 1e9:.3f} GB algorithmic per layer, charged the whole step / 32, input copies, "
     f"allocation and fresh clear included. ncu traffic {k1tr / 1e9:.3f} GB per layer "
     f"(+{(k1tr / r['bytes_per_launch'] - 1) * 100:.0f}%) |",
     f"| same step, batch's blocks randomly permuted over the pool | {fr['value']:.0f} tok/s ({fr['ms_per_step']:.2f} ms) |",
     f"| end to end (pinned host ↔ device every step, {b['e2e']['h2d_bytes_per_step'] / 1e6:.1f} MB H2D + "
     f"{b['e2e']['d2h_bytes_per_step'] / 1e6:.1f} MB D2H) | {b['e2e']['value']:.0f} tok/s |",
     f"| reference arm (`--impl reference`: oracle port on {ref['cpu_baseline']['cores']} host cores) | {ref['value']:.1f} tok/s |",
     f"| eviction per new 32k sequence | K2 {p['k2_window_metric']:.3f} ms + K3/K4 {p['k3k4_schedule_compact']:.3f} ms = {p['total']:.3f} ms |",
     f"| eviction vs one decode step | {e['ratio_to_decode_step']['raw_with_k2'] * 100:.1f}% raw with K2; "
     f"{e['ratio_to_decode_step']['raw_without_k2'] * 100:.1f}% raw without K2; "
     f"{e['ratio_to_decode_step']['amortised_500_tokens_with_k2'] * 100:.2f}% amortised over 500 output tokens |",
     f"| prefill side per sequence (K/V into the cache + metric + compress) | unfused {ps['unfused_scatter_k2_k3k4']:.2f} ms; "
     f"**fused `prefill_compress_sequence` {ps['fused_prefill_compress']:.2f} ms**, less than the plain prompt write "
     f"({p['kv_scatter_not_counted']:.2f} ms) |"]
if mg:
    L.append(f"| on-prefill eviction step, marginal over the plain prompt write | **{mg['ms_per_sequence']:+.2f} ms** "
             f"({mg['ratio_to_decode_step'] * 100:+.1f}% of a decode step) |")
L += [f"| every-step policy: compress() over all 64 sequences | {dr['ms'][-1]:.2f} ms ({dr['ratio_to_decode_step'] * 100:.1f}% of a step) |",
      f"| CPU oracle port, 1 core | decode {b['cpu_baseline']['value']:.1f} tok/s; eviction "
      f"{b['cpu_baseline']['eviction_step_ms_per_sequence'] / 1e3:.1f} s per sequence |\n",
      "## BASELINE configs and the batch sweep (`tools/run_configs.sh` → `profiles/configs/`)\n", cfg,
      "* Small batches are latency-bound: a layer has too little K/V to fill 148 SMs. The CUDA-graph step,",
      "  the batch-sized split-KV items and the parallel partial merge took B=1 from 1.85 to 0.57 ms per step.",
      "* At 128k (Llama-70B shapes), one CTA's score tiles exceed TMEM. K2 therefore streams each layer twice",
      "  (recompute mode).",
      "* At 1x nothing is evicted. The fused path's gather placement is then slower than the plain scatter.\n",
      "## Other paths\n", "| path | measurement | source |", "|---|---|---|",
      f"| KVC-full metric (f3), Llama-8B shapes, one layer at 32k | {f32['ms_per_layer']:.1f} ms, {f32['tflops']:.0f} "
      f"TFLOP/s useful, {f32['gexp_per_s'] / 1e3:.2f} T exp2/s | `profiles/r1_full_metric.json`, `profiles/r1_ncu_full.json` |",
      f"| device Engine (f1) vs reference engine, toy serving workload | {eng['device']['seconds']:.1f} s vs "
      f"{eng['reference_cpu']['seconds']:.1f} s ({eng['reference_cpu']['seconds'] / eng['device']['seconds']:.0f}x), same "
      f"{eng['device']['steps']} steps / {eng['device']['compressions']} compressions | `profiles/r1_engine.json` |\n",
      "## ncu --set full (cold caches, serialised; `profiles/r1_ncu*.json`, recipe `profiles/capture.sh`)\n",
      "| kernel | µs | DRAM read MB | DRAM write MB | GB/s | DRAM % | tcgen05 pipe % |", "|---|---|---|---|---|---|---|"]
for k in ("k1", "k2", "evict", "scatter"):
    L += [row(x) for x in n[k]]
L += [row(x) for x in nf["full"]]
L += ["",
      "* **K1** per layer is `k_decode_stream` + `k_decode_finish` (output merge) + `k_decode_metric`",
      "  (metric accumulation on the graph's side branch, overlapping the next layer).",
      "  * The stream kernel alone runs at ~6.2 TB/s.",
      "  * With the per-block math skipped it streams the same blocks in 163 vs 186 µs, so the math costs",
      "    about 12% (`KVC_K1_TRACE`).",
      "* **K2** (`k_window_persist`, one launch for all 32 layers) reads K exactly once, 2.15 GB per sequence.",
      "  Per layer, its epilogue's serial work is:",
      "  * statistics;",
      "  * a head barrier (~3 µs: skew + latency);",
      "  * the metric pass (~4 µs, it frees the TMEM slots);",
      "  * the previous layer's install (~2 µs).",
      "  That is about as long as the 10 µs stream, so the two alternate rather than overlap.",
      "* **K3** takes about 100 µs: `k_load`, 2 × `k_hist` with the digit finds fused in, `k_bounds`,",
      "  `k_select` and `k_offsets`.",
      "* **K4**: `k_compact16` (latency-bound metadata compaction) takes 110-118 µs, and `k_copy_kv_heads`",
      "  (0.9 GB of K/V moves) about 150 µs.\n",
      "## Read ceiling on this B200 (`tools/microbench/readbw.cu`, 8 GiB buffer)\n",
      "| load path | GB/s |", "|---|---|",
      "| LDG.128, 8 in flight per thread, 4-16 CTAs/SM | 6764-6809 |",
      "| TMA 3-D box {64,16,2} SW128 (K1's block box), 2 CTAs/SM × 4 × 16 KB | 7334 |",
      "| TMA 3-D box {64,128,2} SW128 (K2's tile box), 1 CTA/SM × 4 × 32 KB | 7314 |",
      "| TMA 1-D bulk, 1 CTA/SM × 4 × 32 KB | 7368 |\n",
      "## Progress within the round\n", "| change | before | after |", "|---|---|---|",
      "| K1: warp-independent items, prefetched tables, 2 CTAs/SM | 46% of HBM | 73-80% |",
      "| K1: CUDA-graph decode step; batch-sized split-KV items; parallel partial merge | B=1 1.85 ms/step, B=64 6.89 | B=1 0.57, B=64 6.60 |",
      "| K1: metric on the graph's side branch; ex2.approx; rescale only when a max moved; finish split by batch | B=64 6.60 ms/step | 6.42 |",
      "| K1: finish folds the C bump and queue reset, pre-wait loads, float4 merge | B=64 6.42 ms/step; l70b 10.0 | 6.24; 9.50 |",
      "| K1: scores and partials stored L2 evict_last, discarded by their readers (never written back) | B=64 6.24 ms/step; l70b 9.50 | 6.02; 8.80 |",
      "| K1: first work-item pull and TMA loads before griddepcontrol.wait (alternating queue heads) | 10.78k tok/s | 10.87k tok/s (same box) |",
      "| K0: k_decode_demand with 16 heads per thread (independent C loads, one scan per tile) | 26 us/step | 19 us/step |",
      "| e2e: per-layer host upload/download inside the graph (`host_io`), uploads awaited per doubling layer group | e2e 9.1k tok/s | 10.6k |",
      "| K2: persistent multi-layer kernel (TMEM slot ring across layers, one barrier per layer, branch-free ex2) | 1.39-1.48 ms/seq | 0.52 ms/seq |",
      "| K2: recompute mode at 128k | 33.5 ms/seq (two-pass fallback) | 7.7 ms/seq |",
      "| K2: head barrier as red.release + ld.acquire poll instead of two fence.sc (its top stall in ncu) | 0.52 ms/seq | 0.48 ms/seq |",
      "| K4: 512-thread compaction CTAs, aggregated free-tile atomics, batched metadata moves | K3+K4 0.48 ms | 0.38 ms |",
      "| K4: one-pass tie cut in shared memory; threshold select started at T*'s top digit bins | K3+K4 0.385 ms | 0.352 ms |",
      "| prompt scatter: warp-per-block, multi-layer kernel | 2.9 ms/seq | 1.37 ms/seq |",
      "| fused prefill + compress (survivors written once) | 2.30 ms/seq | 1.15 ms/seq |",
      f"| KVC-full: 8 epilogue warps, chunk-max softmax, pre-multiplied normalisers, 2 CTAs/SM | 16.8 ms/layer (32k) | {f32['ms_per_layer']:.1f} |",
      "\nExperiments that were measured and dropped:",
      "* K1: eager side-stream metric (broke the PDL chain); L2 prefetch ahead of the ring (slower at every",
      "  distance); tail-split items; smaller items at large B (8-block items: l8b 9.9k vs 10.6k tok/s, after the",
      "  L2-resident partials); packed score stores; a producer warp per CTA that pre-fetches each warp's next",
      "  item and query rows into shared memory (l8b 10.5k, l70b 7.07k, m7b 18.3k vs 10.6k / 7.27k / 19.5k);",
      "  each head's last chunk as four quarter items queued last (l8b 10.4k vs 10.7k, m7b 18.1k vs 19.4k): while",
      "  the queue drains, the warps still streaming keep HBM saturated, so the warps' end-time spread costs less",
      "  than the extra items do.",
      "* K2:",
      "  * pipelined metric pass;",
      "  * L2 prefetch ahead of the ring;",
      "  * recompute mode at 32k (20.5 vs 15.4 µs/layer);",
      "  * two score tiles parked in smem (16.0 vs 15.4 µs/layer);",
      "  * split head barrier with the previous layer's install between arrive and wait (0.635 vs 0.52 ms/seq).",
      "* K4: PDL-overlapped K/V copy; the copy inside the compaction warps; unrolled and warp-aggregated or",
      "  privatised histogram atomics in the selects; pipelined survivor pass.",
      "* KVC-full: 30% of the exp2s as an FMA polynomial. The epilogue is issue-bound, so it was slower.",
      "* K2: spinning without `nanosleep` in the head barrier poll (0.479 vs 0.478 ms/seq).",
      "* K4: the same one-pass tie cut in the warp-per-head `k_compact_warp` (decode-round compress 1.105 vs",
      "  1.04 ms: ties are rare on that path).",
      "* K1: 8-byte packed score stores (full sectors) with the L2-resident scores: l8b +0.3%, l70b -0.7%,",
      "  m7b -0.5%; per-block score staging in shared memory written by one `cp.async.bulk` store (l8b 10.5k vs",
      "  10.7k: the per-block proxy fence and bulk-group wait cost more than the four stores).",
      "",
      "Where the decode metric's 5.5% goes (ncu `--graph-profiling graph`, one whole step): it adds only",
      "0.81 GB of DRAM traffic per step. That is the 16.8 MB/layer metric read-modify-write plus ~8 MB/layer",
      "of score lines that leave L2, so the 33.5 MB/layer score rows mostly stay in L2. The time goes to the",
      "score stores themselves: with the metric off, forcing the stores costs 0.29 ms of the 0.39 ms.",
      "* K3: 8 uint4 key loads in flight in `k_hist` (60 registers halved its occupancy; decode round 1.16 vs",
      "  1.06 ms); kept in `k_bounds`' long-head path, where registers went down.",
      "",
      "K4 select shortcut: `k_bounds` now also counts, per head, the keys below T* that share T*'s top",
      "11/22 bits. `k_compact16` then starts its per-head threshold select at level 2 or 3 (per-head",
      "threshold phase 22.0 -> 17.6 us; per-sequence K3+K4 unchanged within noise, since later passes hit L2).",
      "K4 tie cut: the pooled window metric repeats a local maximum over neighbouring slots, so the cut",
      "inside the ties at the threshold runs for every head. With <= 512 ties, `k_compact16` now collects",
      "their secondary keys in one pass and ranks them in shared memory instead of three radix passes: tie",
      "phase 23 -> 4.5 us per head, compaction span 107 -> 83 us, K3+K4 0.377 -> 0.352 ms per sequence."]
open(os.path.join(HERE, "r1_summary.md"), "w").write("\n".join(L) + "\n")
