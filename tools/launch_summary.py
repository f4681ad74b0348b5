"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel: launches, mean
duration and share of device time.

    python tools/launch_summary.py launches.csv
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, defaultdict(list)
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        iK, iM, iV, iU = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
        continue
    if hdr and len(r) > iV and r[iM] == "gpu__time_duration.sum":
        agg[r[iK][:70]].append(float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0))
tot = sum(sum(v) for v in agg.values())
print("# Launch list of `python bench.py --steps 5 --warmup 3 --no-cpu-baseline` (C2) under")
print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES).")
print("# kernel | launches | mean ms | share of device time")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k} | {len(v)} | {sum(v) / len(v):.4f} | {100 * sum(v) / tot:.1f}%")
