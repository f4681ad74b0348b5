"""Print the round-2 bench table (profiles/r2/bench_*_final.json) for DESIGN.md / README."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
print("| Config | Points | Step (ms) | Request-iterations/s | e2e (C ABI, host buffers) | Oracle (16 cores) | x oracle |")
print("|---|---|---|---|---|---|---|")
for c in ("c1", "c2", "c3", "c4", "c5", "c6", "c7", "c8", "c9"):
    p = os.path.join(ROOT, "profiles", "r2", f"bench_{c}_final.json")
    if not os.path.exists(p):
        continue
    d = json.loads(open(p).read().strip().splitlines()[-1])
    cb = d.get("cpu_baseline") or {}
    ov = cb.get("value") or 0
    print(f"| {c.upper()} | {d['config']['points']} | {d['ms_per_step']:.1f} | {d['value']:.3g} | {d['e2e']['value']:.3g} | "
          f"{ov:.3g} | {d['value'] / ov:.0f} |" if ov else f"| {c} | ... |")
