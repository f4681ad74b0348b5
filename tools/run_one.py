"""Run one point of a preset alone (one CTA) on cuda:0 -- a minimal target for ncu captures.

    python tools/run_one.py --config c6 --point 7
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import sweep_inputs as si  # noqa: E402
import paper_2503_08415_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c6")
ap.add_argument("--point", type=int, default=7)
a = ap.parse_args()
sw = P.Sweep(si.PRESETS[a.config]())
sw.run(a.point, a.point + 1, 1)
torch.cuda.synchronize()
info = sw.run_info()
print(a.config, "point", a.point, "sim ms %.2f" % info["ms_sim"], "iters", int(sw.summaries()["n_iterations"][0]))
