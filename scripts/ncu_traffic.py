"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
and duration for each kernel in an ncu report into profiles/ncu_traffic.json
(bench.py reports it as roofline.traffic for the matching kernel)."""
import csv
import json
import os
import subprocess
import sys

out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "ncu_traffic.json")
db = json.load(open(out_path)) if os.path.exists(out_path) else {}
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]

    def val(row, m):
        i = h.index(m)
        v = float(row[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
                 "usecond": 1, "msecond": 1e3}.get(u, 1)
        return v * scale

    for row in rows[2:]:
        name = row[h.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").strip()
        rd = val(row, "dram__bytes_read.sum")
        wr = val(row, "dram__bytes_write.sum")
        dur = val(row, "gpu__time_duration.sum")
        db[name] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                    "duration_us_cold": dur, "report": os.path.basename(rep)}
json.dump(db, open(out_path, "w"), indent=1, sort_keys=True)
print(json.dumps(db, indent=1))
