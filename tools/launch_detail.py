"""Per-kernel, per-grid-size summary of an ncu launch list (dev tool)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")   # ncu prints warnings first
rows = rows[start:]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
gi = h.index("Grid Size") if "Grid Size" in h else None
agg = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    g = r[gi] if gi is not None else ""
    agg[name].append((float(r[vi].replace(",", "")), g))
for name, v in sorted(agg.items(), key=lambda x: -sum(t for t, _ in x[1])):
    ts = sorted(t for t, _ in v)
    print(f"{name:20s} n={len(v):5d} total={sum(ts)/1e3:9.1f}us  min={ts[0]/1e3:7.1f} med={ts[len(ts)//2]/1e3:7.1f} max={ts[-1]/1e3:8.1f}")
    by = collections.defaultdict(list)
    for t, g in v:
        by[g].append(t)
    for g, tt in sorted(by.items(), key=lambda x: -sum(x[1]))[:4]:
        print(f"     grid {g:>18s}: n={len(tt):4d} avg={sum(tt)/len(tt)/1e3:7.1f}us")
