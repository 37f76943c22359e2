"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes):
one line per launch of the package's kernels.  usage: launch_table.py CSV [regex]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else r"ctkv|tc::")
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr, start = r, i + 1
        break
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[start:]:
    if len(r) > vi:
        agg.setdefault((int(r[0]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
for (i, k), d in agg.items():
    if pat.search(k):
        print(f"{i:6d} {k[:64]:64s} {d.get('gpu__time_duration.sum', 0) / 1e3:10.1f} us "
              f"{d.get('dram__bytes_read.sum', 0) / 1e6:9.1f} MB r {d.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB w")
