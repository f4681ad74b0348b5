"""Minimal driver for ncu captures: one sweep run of a preset on cuda:0.

    python tools/prof_run.py --config c2 [--reps 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import sweep_inputs as si  # noqa: E402
import paper_2503_08415_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--points", type=int, default=0, help="run only the first N points")
a = ap.parse_args()
cfg = si.PRESETS[a.config]()
sw = P.Sweep(cfg)
end = a.points or sw.num_points
for _ in range(a.reps):
    sw.run(0, end, 1)
    torch.cuda.synchronize()
    info = sw.run_info()
    s = sw.summaries()
    print(a.config, "points", len(s), "req-its", int(s["n_request_iterations"].sum()),
          "iters max", int(s["n_iterations"].max()), "sim ms %.3f" % info["ms_sim"],
          "grid", info["sim_blocks"], "x", info["sim_warps_per_block"], "smem/warp", info["smem_per_warp"])
