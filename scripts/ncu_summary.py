"""Key ncu metrics per kernel from an .ncu-rep (details page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Achieved Occupancy", "Registers Per Thread", "Issue Slots Busy", "No Eligible",
        "L2 Hit Rate", "Grid Size", "Dynamic Shared Memory Per Block", "Executed Ipc Active"]
seen = set()
for r in rows[1:]:
    key = (r[ki], r[mi])
    if r[mi] in want and key not in seen:
        seen.add(key)
        print(f"- {r[ki].split('(')[0][:60]} | {r[mi]}: {r[vi]} {r[ui]}")
