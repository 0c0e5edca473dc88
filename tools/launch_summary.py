"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0,
             "msecond": 1.0}.get(r[ui], 1e-6)
    name = r[ki][:70]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v * scale
tot = sum(a[1] for a in agg.values())
print("| kernel | launches | total ms | ms/launch | share |\n|---|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {n} | {t:.3f} | {t / n:.4f} | {100 * t / tot:.2f} % |")
