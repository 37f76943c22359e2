"""Top SASS instructions by warp-stall samples from
`ncu -i REP --page source --csv --print-source sass` (with the dominant stall reasons)."""
import csv
import sys

path, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path, errors="replace")))
h = rows[1]
data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
tot = sum(float(r[si] or 0) for r in data if len(r) > si) or 1
print(f"total samples {tot:.0f}")
agg = {}
for i in stall_cols:
    agg[h[i]] = sum(float(r[i] or 0) for r in data if len(r) > i and r[i] not in ("", "-"))
print("stall totals:", ", ".join(f"{k[6:]}={100*v/tot:.1f}%" for k, v in
                                  sorted(agg.items(), key=lambda x: -x[1])[:8]))
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
    s = float(r[si] or 0)
    top = sorted(((float(r[i] or 0) if r[i] not in ("", "-") else 0, h[i][6:]) for i in stall_cols),
                 reverse=True)[:2]
    print(f"{s:7.0f} {100*s/tot:5.1f}% {r[0]:>6} {r[1][:60]:60s} " +
          " ".join(f"{k}:{v:.0f}" for v, k in top))
