"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv --log-file X` launch list into a markdown table:
per (kernel, grid) the launch count, mean duration and mean DRAM traffic."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
rows = [r for r in csv.reader(open(path, errors="replace")) if r]
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ki, gi, mi, vi, idi = (h.index(x) for x in ("Kernel Name", "Grid Size", "Metric Name", "Metric Value", "ID"))
per = defaultdict(dict)
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    try:
        per[(r[idi], r[ki], r[gi])][r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        pass
agg = defaultdict(lambda: [0, 0.0, 0.0])
for (_, k, g), m in per.items():
    name = k.split("(")[0].replace("void ", "")
    a = agg[(name, g)]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
unit_t = 1e-3   # ncu reports ns for gpu__time_duration.sum in csv; convert to us
print("| kernel | grid | launches | mean us | mean DRAM MB/launch |")
print("|---|---|---|---|---|")
for (name, g), (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {name} | {g} | {n} | {t / n * unit_t:.1f} | {b / n / 1e6:.1f} |")
