"""Epoch profile of the xP:yD node kernel (sim_pdn.cuh) on a preset (default c6).

    python tools/node_prof.py [--config c6] [--top 6]

Prints, for the longest points: SM cycles, iterations, epochs, and the cycles warp 0 spent in
scheduler phases, its own decode phases, and the largest / summed decode-phase cycles over the
decode warps, its horizon computations and its waits for the slowest decode warp
(point_profile's stretch_phase_cycles[0..6] for node points).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import sweep_inputs as si  # noqa: E402
import paper_2503_08415_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c6")
ap.add_argument("--top", type=int, default=6)
a = ap.parse_args()
cfg = si.PRESETS[a.config]()
sw = P.Sweep(cfg)
sw.run()
torch.cuda.synchronize()
info = sw.run_info()
print(a.config, "sim ms %.2f" % info["ms_sim"], "grid", info["sim_blocks"], "x", info["sim_warps_per_block"])
prof = [sw.point_profile(p) for p in range(sw.num_points)]
cy = np.array([x["sm_cycles"] for x in prof], dtype=np.float64)
for p in np.argsort(-cy)[:a.top]:
    x = prof[p]
    ph = x["stretch_phase_cycles"]
    print(f"point {p}: cycles {x['sm_cycles']:.3e} iters {x['n_iterations']} ff {x['ff_iterations']} "
          f"stretches {x['ff_stretches']} epochs {ph[0]} sched {ph[1]:.3e} dec0 {ph[2]:.3e} "
          f"dec_max {ph[3]:.3e} dec_sum {ph[4]:.3e} horizon {ph[5]:.3e} wait {ph[6]:.3e} "
          f"cyc/epoch {x['sm_cycles'] / max(1, ph[0]):.0f}")
ms = cy / 1.965e6
q = np.percentile(ms, [0, 10, 25, 50, 75, 90, 100])
print("per-point ms at 1.965 GHz: min/p10/p25/p50/p75/p90/max", " ".join("%.0f" % v for v in q),
      "| sum / SMs %.0f ms" % (ms.sum() / 148))
