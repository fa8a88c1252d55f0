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


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
