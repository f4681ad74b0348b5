"""A/B of the LPT order: the a-priori cost estimate vs the measured per-point costs (an upper
bound for what a better estimate could give).  One GPU:

    python tools/lpt_exp.py --config c3
"""
import argparse
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

CHILD = r"""
import os, sys, json
sys.path.insert(0, %(root)r)
import numpy as np, torch, sweep_inputs as si, paper_2503_08415_b200 as P
cfg = si.PRESETS[%(cfg)r]()
sw = P.Sweep(cfg)
best = 1e30
for r in range(%(reps)d + 1):
    sw.run()
    torch.cuda.synchronize()
    ms = sw.run_info()["ms_sim"]
    if r: best = min(best, ms)
out = os.environ.get("DUMP")
if out:
    c = np.array([sw.point_profile(p)["sm_cycles"] for p in range(sw.num_points)], dtype=np.float64)
    c.tofile(out)
print(json.dumps({"ms_sim": best}))
"""
src = CHILD % {"root": ROOT, "cfg": a.config, "reps": a.reps}
costs = "/tmp/lpt_costs.bin"
r1 = subprocess.run([sys.executable, "-c", src], env=dict(os.environ, DUMP=costs), capture_output=True, text=True)
print("estimate order:", r1.stdout.strip(), r1.stderr[-300:])
r2 = subprocess.run([sys.executable, "-c", src], env=dict(os.environ, TOKENSIM_LPT_COSTS=costs), capture_output=True,
                    text=True)
print("measured-cost order:", r2.stdout.strip(), r2.stderr[-300:])
