"""A/B helper: one C3-shaped sweep with small per-warp shared memory (capacities <= 80 GB), timed
with the library named by TOKENSIM_LIB (used to compare register/occupancy trade-offs)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import sweep_inputs as si  # noqa: E402
import paper_2503_08415_b200 as P  # noqa: E402

base = si.c3()
caps = [i for i, h in enumerate(base.hws) if h.mem_capacity <= 80e9]
cfg = si.subset(base, hws=caps)
sw = P.Sweep(cfg)
best = 1e30
for _ in range(3):
    sw.run()
    torch.cuda.synchronize()
    info = sw.run_info()
    best = min(best, info["ms_sim"])
s = sw.summaries()
print(os.environ.get("TOKENSIM_LIB", "default"), "points", len(s), "req-its", int(s["n_request_iterations"].sum()),
      "sim ms %.1f" % best, "grid", info["sim_blocks"], "x", info["sim_warps_per_block"], "smem/warp", info["smem_per_warp"],
      "req-it/s %.3e" % (s["n_request_iterations"].sum() / best * 1e3))
