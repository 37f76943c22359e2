"""Summarise an `ncu --page source --print-source cuda,sass --csv` dump:
warp-stall samples per CUDA source line (file:line), top N."""
import csv
import sys
from collections import defaultdict

path, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
agg = defaultdict(float)
text = {}
cur_file, cur_line = "?", None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 6 or r[0] == "Line No":
        continue
    if r[0] not in ("", "-"):
        cur_line = r[0]
        text[(cur_file, cur_line)] = r[1].strip()
        try:
            agg[(cur_file, cur_line)] += float(r[4])
        except ValueError:
            pass
tot = sum(agg.values()) or 1
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    print(f"{v:8.0f} {100*v/tot:5.1f}%  {f}:{l}  {text.get((f,l),'')[:90]}")
