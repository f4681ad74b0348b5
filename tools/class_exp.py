"""A/B of the point-queue order on C3 by code-path class: LPT by measured per-point cost vs the
same costs with the queue grouped by policy kind, and by KV capacity class -- grouping puts
warps that run the same code paths on the GPU at the same time (the 8-warps-per-SM kernel is
instruction-fetch bound).  One GPU:

    python tools/class_exp.py
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys, json
sys.path.insert(0, %(root)r)
import numpy as np, torch, sweep_inputs as si, paper_2503_08415_b200 as P
cfg = si.PRESETS["c3"]()
sw = P.Sweep(cfg)
best = 1e30
h = None
for r in range(4):
    sw.run()
    torch.cuda.synchronize()
    ms = sw.run_info()["ms_sim"]
    if r: best = min(best, ms)
out = os.environ.get("DUMP")
if out:
    c = np.array([sw.point_profile(p)["sm_cycles"] for p in range(sw.num_points)], dtype=np.float64)
    c.tofile(out)
import hashlib
print(json.dumps({"ms_sim": best, "hash": hashlib.sha256(sw.summaries().tobytes()).hexdigest()[:16]}))
"""


def run(env):
    r = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT}], env=dict(os.environ, **env),
                       capture_output=True, text=True)
    return r.stdout.strip() or r.stderr[-400:]


costs = "/tmp/c3_costs.bin"
print("estimate order:", run({"DUMP": costs}))
c = np.fromfile(costs, dtype=np.float64)
p = np.arange(len(c))
pol, hw = p % 3, p // 3
cap = hw % 6
print("measured-cost order:", run({"TOKENSIM_LPT_COSTS": costs}))
for name, key in (("grouped by policy", 2 - pol), ("grouped by capacity", 5 - cap),
                  ("grouped by capacity, small first", cap)):
    f = f"/tmp/c3_costs_{name.replace(' ', '_').replace(',', '')}.bin"
    (key.astype(np.float64) * 1e15 + c).tofile(f)
    print(name + ":", run({"TOKENSIM_LPT_COSTS": f}))
