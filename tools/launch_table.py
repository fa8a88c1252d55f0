"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: mean us per kernel name."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
acc = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] in ("ns", "nsecond") else v * 1e3 if r[ui] in ("ms", "msecond") else v
    acc.setdefault(name, []).append(v)
for k, v in acc.items():
    print(f"{k:40s} n={len(v):4d} mean={sum(v)/len(v):9.1f} us  min={min(v):9.1f}")
