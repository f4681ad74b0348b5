"""Split an ncu source page (--print-source=cuda,sass CSV) into the helper warp's and the
simulating warp's shares, by SASS address range of helper_loop (one-warp-per-SM kernel).

    python tools/ncu_split.py x.csv HELPER_FIRST_LINE HELPER_LAST_LINE [topN]
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
h0, h1 = int(sys.argv[2]), int(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
hdr = None
cur_file, cur_line, cur_src = "?", 0, ""
sass = []  # (addr, file, line, src, samples, instr)
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
        continue
    if r[2].startswith("0x"):
        sass.append((int(r[2], 16), cur_file, cur_line, cur_src, num(r[i_s]), num(r[i_ie])))
# owner of each SASS row: the nearest sim_core.cuh row at or before it in address order decides
# (inlined helpers from other files inherit the owner of the code they were inlined into)
sass.sort()
owner, cur = {}, "simulating"
for a, f, l, *_ in sass:
    if f.startswith("sim_core"):
        cur = "helper" if h0 <= l <= h1 else "simulating"
    owner[a] = cur
tot = sum(x[4] for x in sass)
for name in ("helper", "simulating"):
    part = [x for x in sass if owner[x[0]] == name]
    s = sum(x[4] for x in part)
    print(f"{name}: {s} stall samples ({100 * s / max(1, tot):.1f}%), {sum(x[5] for x in part)} warp instructions")
    agg = defaultdict(lambda: [0, 0, ""])
    for a, f, l, src, st, ie in part:
        g = agg[(f, l)]
        g[0] += st
        g[1] += ie
        g[2] = src
    for (f, l), (st, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {f[:10]:10s}{l:5d} {100 * st / max(1, s):5.1f}% {ie:10d}  {src.strip()[:90]}")
