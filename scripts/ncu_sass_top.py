"""Top SASS instructions by warp-stall samples from
`ncu -i REP --page source --csv --print-source sass [-k NAME]` (with the
dominant stall reasons).  Handles multi-kernel dumps: only the first
kernel's table is read."""
import csv
import sys

path, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path, errors="replace")))
start = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[start]
data = []
for r in rows[start + 1:]:
    if r and r[0] in ("Address", "Kernel Name"):
        break
    data.append(r)
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(num(r[si]) for r in data if len(r) > si) or 1
print(f"total samples {tot:.0f}")
agg = {h[i]: sum(num(r[i]) for r in data if len(r) > i) for i in stall_cols}
print("stall totals:", ", ".join(f"{k[6:]}={100*v/tot:.1f}%" for k, v in
                                  sorted(agg.items(), key=lambda x: -x[1])[:8]))
for r in sorted(data, key=lambda r: -num(r[si]))[:n]:
    s = num(r[si])
    top = sorted(((num(r[i]), h[i][6:]) for i in stall_cols), reverse=True)[:2]
    print(f"{s:7.0f} {100*s/tot:5.1f}% {r[0][-5:]:>6} {r[1][:64]:64s} " +
          " ".join(f"{k}:{v:.0f}" for v, k in top))
