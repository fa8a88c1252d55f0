"""Markdown table of the bench.py config runs (profiles/configs/*.json)."""
import glob
import json
import os
import sys

root = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "profiles", "configs")
rows = []
for f in sorted(glob.glob(os.path.join(root, "*.json"))):
    try:
        d = json.load(open(f))
    except Exception:
        continue
    c, e = d["config"], d["eviction_step"]
    rows.append((c["preset"], c["batch_per_gpu"], c["compression"], d["value"], d["ms_per_step"], d["roofline"]["frac"],
                 e["per_sequence_ms"]["k2_window_metric"], e["per_sequence_ms"]["k3k4_schedule_compact"],
                 e["prefill_side_per_sequence_ms"]["unfused_scatter_k2_k3k4"],
                 e["prefill_side_per_sequence_ms"]["fused_prefill_compress"],
                 e["ratio_to_decode_step"]["raw_with_k2"], e["ratio_to_decode_step"]["raw_without_k2"],
                 e["ratio_to_decode_step"]["amortised_500_tokens_with_k2"], os.path.basename(f)))
order = {"toy": 0, "l8b": 1, "m7b": 2, "l70b": 3}
rows.sort(key=lambda r: (order.get(r[0], 9), r[2], r[1]))
print("| config | B/GPU | rate | decode tok/s | ms/step | K1 % of HBM | K2 ms/seq | K3+K4 ms/seq | prefill side unfused / fused ms | evict / step raw (with K2 / without) | amortised 500 tok | file |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r[0]} | {r[1]} | {r[2]} | {r[3]:,.0f} | {r[4]:.3f} | {r[5]*100:.1f}% | {r[6]:.3f} | {r[7]:.3f} | {r[8]:.2f} / {r[9]:.2f} | "
          f"{r[10]*100:.1f}% / {r[11]*100:.1f}% | {r[12]*100:.2f}% | `{r[13]}` |")
