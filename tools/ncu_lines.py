"""Aggregate an ncu source page (--print-source=cuda,sass CSV) by CUDA source line.

    ncu -i rep --page source --csv --print-source=cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [topN]
"""
import csv
import os
import sys
from collections import defaultdict


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0, 0, ""])
hdr = None
cur_file, cur_line, cur_src = "?", None, ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or r[0] == "Function Name" or len(r) < len(hdr):
        continue
    if r[0]:
        cur_line, cur_src = num(r[0]), r[1]
    if r[2]:
        a = agg[(cur_file, cur_line)]
        a[0] += num(r[i_s])
        a[1] += num(r[i_ie])
        a[2] = cur_src
tot_s = sum(v[0] for v in agg.values())
tot_i = sum(v[1] for v in agg.values())
print(f"total stall samples {tot_s}, warp instructions executed {tot_i}")
for (f, line), (s, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f[:10]:10s}{line:5d} {100*s/max(1,tot_s):5.1f}% {100*ie/max(1,tot_i):5.1f}%  {src.strip()[:95]}")
