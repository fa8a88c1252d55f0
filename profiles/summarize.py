"""Summarise ncu captures into profiles/ (run in the build container).

    python profiles/summarize.py launches <launches.csv>
    python profiles/summarize.py report <file.ncu-rep>
"""

import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:60]
        tot[name] += float(d["Metric Value"].replace(",", ""))
        cnt[name] += 1
    all_t = sum(tot.values())
    print(f"| kernel | launches | total us | share |\n|---|---|---|---|")
    for name, t in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{name}` | {cnt[name]} | {t / 1e3:.1f} | {t / all_t * 100:.1f}% |")


KEYS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("dram__bytes_read.sum", "DRAM read (B)"),
    ("dram__bytes_write.sum", "DRAM write (B)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (HMMA) %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (tcgen05) %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        name = d.get("Kernel Name", "?").split("(")[0][:48]
        cells = [d.get(k[0], "n/a") for k in KEYS]
        print(f"| `{name}` | " + " | ".join(cells) + " |")


if __name__ == "__main__" and sys.argv[1] != "json":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])


def raw_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))

        def num(key, scale_units):
            v = float(d[key].replace(",", ""))
            return v * scale_units.get(u.get(key, ""), 1.0)

        res.append({
            "kernel": d["Kernel Name"].split("(")[0].replace("<unnamed>::", ""),
            "duration_us": num("gpu__time_duration.sum", {"ns": 1e-3, "us": 1.0, "ms": 1e3}),
            "dram_read_B": num("dram__bytes_read.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
            "dram_write_B": num("dram__bytes_write.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
            "dram_pct_of_peak": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
            "tcgen05_pipe_pct": d.get("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "n/a"),
            "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
            "registers": d.get("launch__registers_per_thread"),
        })
    return res


def to_json(out_path, *pairs):
    """python profiles/summarize.py json profiles/r1_ncu.json k1=prof_k1.ncu-rep k2=... (first launch of each
    kernel name per group)."""
    import json
    doc = {"source": "ncu --set full --clock-control none, cold caches, serialised (profiles/capture.sh)"}
    for pair in pairs:
        key, path = pair.split("=", 1)
        seen, keep = set(), []
        for r in raw_rows(path):
            if r["kernel"] in seen:
                continue
            seen.add(r["kernel"])
            keep.append(r)
        doc[key] = keep
    with open(out_path, "w") as fh:
        json.dump(doc, fh, indent=1)


if __name__ == "__main__" and sys.argv[1] == "json":
    to_json(sys.argv[2], *sys.argv[3:])
