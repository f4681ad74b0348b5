"""Instruction-cache footprint of a kernel from an ncu source page (--print-source=cuda,sass CSV):
executed SASS instructions by 128-B line, and the bytes of lines (vs of instructions) needed to
cover 90 / 95 / 99% of executions.  Also lists the hottest lines' cold neighbours.

    python tools/ncu_icache.py x.csv
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
ins = {}
for r in rows:
    if not r:
        continue
    if r[0] == "Line No":
        hdr = r
        i_ie = hdr.index("Instructions Executed")
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_ni = hdr.index("Warp Stall Sampling (Not-issued Samples)") if "Warp Stall Sampling (Not-issued Samples)" in hdr else None
        continue
    if hdr is None or len(r) < len(hdr) or not r[2].startswith("0x"):
        continue
    a = int(r[2], 16)
    ie = int(r[i_ie]) if r[i_ie].isdigit() else 0
    ins[a] = ins.get(a, 0) + ie
tot = sum(ins.values())
base = min(ins)
lines = defaultdict(int)
for a, ie in ins.items():
    lines[(a - base) // 128] += ie
print(f"instructions {len(ins)} ({16 * len(ins) / 1024:.0f} KB), executed {tot:.3e}")
for frac in (0.9, 0.95, 0.99, 0.999):
    acc, n_ins = 0, 0
    for a, ie in sorted(ins.items(), key=lambda kv: -kv[1]):
        acc += ie
        n_ins += 1
        if acc >= frac * tot:
            break
    acc, n_ln = 0, 0
    for ln, ie in sorted(lines.items(), key=lambda kv: -kv[1]):
        acc += ie
        n_ln += 1
        if acc >= frac * tot:
            break
    print(f"{100 * frac:5.1f}% of executions: {n_ins} instructions = {16 * n_ins / 1024:.1f} KB; "
          f"{n_ln} lines = {128 * n_ln / 1024:.1f} KB")
