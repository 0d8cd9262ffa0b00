"""Share of device time per kernel from an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launch_list_summary.txt
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    name = name.replace("void ", "")
    name = name.split("<")[0]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
all_us = sum(tot.values())
print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches;")
print("# compare shares, not absolutes).  Command: " + (sys.argv[2] if len(sys.argv) > 2 else "see DESIGN.md"))
for name, us in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{name:48s} launches {cnt[name]:5d}  total_us {us:12.1f}  share {100 * us / all_us:5.1f}%")
