"""Markdown table of the bench lines in profiles/<round>/bench_*.json."""
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "profiles/r1"
names = [("default", "C2 (default)"), ("c3", "C3"), ("c4", "C4"), ("c5", "C5 (one seed / GPU)"),
         ("c6", "c6 NEXT-1 P2:D6 node"), ("c7", "c7 NEXT-2 multi-round + cache"),
         ("c8", "c8 NEXT-3 MIXED / PF / CHUNKED"), ("c9", "c9 NEXT-4 preload link")]
print("| Config | Points | Step (ms) | Request-iterations/s | e2e (C ABI, host buffers) | Oracle (16 cores) | ×oracle |")
print("|---|---|---|---|---|---|---|")
for f, label in names:
    p = os.path.join(d, f"bench_{f}.json")
    if not os.path.exists(p):
        continue
    b = json.load(open(p))
    cb = b.get("cpu_baseline") or {}
    ratio = b["value"] / cb["value"] if cb.get("value") else None
    print(f"| {label} | {b['config'].get('points')} | {b['ms_per_step']:.1f} | {b['value']:.3g} | "
          f"{b['e2e']['value']:.3g} | {cb.get('value', float('nan')):.3g} | {ratio:.0f} |" if ratio else
          f"| {label} | {b['config'].get('points')} | {b['ms_per_step']:.1f} | {b['value']:.3g} | "
          f"{b['e2e']['value']:.3g} | (reference arm) | |")
