"""Top SASS lines of an ncu source-page CSV (--page source --csv --print-source sass) by warp
stall samples, with the dominant stall reasons of each line.
usage: python tools/ncu_src_top.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


tot = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
print(f"total samples {tot:.0f}")
agg = {c: sum(num(d[c]) for d in data) for c in stall_cols}
print("by reason:", ", ".join(f"{c[6:]} {v / tot:.1%}" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
data.sort(key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))
for d in data[:n]:
    s = num(d["Warp Stall Sampling (All Samples)"])
    top = sorted(((num(d[c]), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{d['Address']:>6} {s / tot:6.1%}  {d['Source'][:60]:60s} " +
          " ".join(f"{c}:{v:.0f}" for v, c in top if v))
