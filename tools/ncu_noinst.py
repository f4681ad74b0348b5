"""Instruction-fetch view of an ncu source page (--print-source=cuda,sass CSV): per source line,
the distinct SASS instructions executed, the executions, all stall samples and the
no-instruction (instruction-cache miss) stall samples.

    python tools/ncu_noinst.py x.csv [topN]
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
hdr = None
fil = "?"
cur = None
per = defaultdict(lambda: [set(), 0, 0, 0])
addr_exec = {}
for r in rows:
    if r and r[0] == "File Path":
        fil = os.path.basename(r[1])
        continue
    if r and r[0] == "Line No":
        hdr = r
        i_ie, i_ni, i_s = hdr.index("Instructions Executed"), hdr.index("stall_no_inst"), hdr.index(
            "Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r or len(r) < len(hdr) or r[0] == "Function Name":
        continue
    if r[0]:
        cur = (fil, num(r[0]), r[1].strip()[:80])
    if r[2]:
        a = per[cur]
        if num(r[i_ie]) > 0:
            a[0].add(r[2])
        a[1] += num(r[i_ie])
        a[2] += num(r[i_s])
        a[3] += num(r[i_ni])
        addr_exec[r[2]] = addr_exec.get(r[2], 0) + num(r[i_ie])
S = sum(v[2] for v in per.values())
NI = sum(v[3] for v in per.values())
E = sum(addr_exec.values())
vals = sorted(addr_exec.values(), reverse=True)
acc, k90, k99 = 0, 0, 0
for i, x in enumerate(vals):
    acc += x
    if not k90 and acc >= 0.9 * E:
        k90 = i + 1
    if acc >= 0.99 * E:
        k99 = i + 1
        break
print(f"stall samples {S}, no-instruction {NI} ({100 * NI / max(1, S):.1f}%); executed SASS {sum(1 for v in vals if v)}"
      f" distinct, 90% of executions in {k90} ({k90 * 16 // 1024} KB), 99% in {k99} ({k99 * 16 // 1024} KB)")
print(" no-inst%  all%  distinct  source")
for k, v in sorted(per.items(), key=lambda kv: -kv[1][3])[:top]:
    print(f"{100 * v[3] / max(1, NI):7.1f} {100 * v[2] / max(1, S):5.1f} {len(v[0]):6d}   {k[0][:12]:12s}{k[1]:5d} {k[2]}")
