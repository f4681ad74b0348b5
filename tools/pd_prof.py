"""Cycle split of a P/D sweep (1P:1D pair): D fast-forward / failed attempts / D normal / rest."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if not os.environ.get("TOKENSIM_LIB"):  # the cycle splits need the profiling build
    import importlib.util  # load build.py alone: importing the package would load the product library
    _spec = importlib.util.spec_from_file_location(
        "ts_build", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2503_08415_b200",
                                 "build.py"))
    _b = importlib.util.module_from_spec(_spec)
    _spec.loader.exec_module(_b)
    os.environ["TOKENSIM_LIB"] = _b.build_profiling()
import numpy as np  # noqa: E402
import torch  # noqa: E402
import sweep_inputs as si  # noqa: E402
import paper_2503_08415_b200 as P  # noqa: E402

cfg = si.PRESETS[sys.argv[1] if len(sys.argv) > 1 else "c5"]()
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
sw = P.Sweep(cfg)
sw.run(0, min(n, sw.num_points), 1)
torch.cuda.synchronize()
prof = [sw.point_profile(p) for p in range(min(n, sw.num_points))]
tot = np.array([[x["sm_cycles"], x["cycles_ff"], x["cycles_ff_failed"], x["cycles_normal"], x["n_iterations"],
                 x["ff_iterations"], x["ff_stretches"], x["n_transfers"]] for x in prof], dtype=np.float64).sum(0)
s = sw.summaries()
print("points", len(prof), "sim ms %.1f" % sw.run_info()["ms_sim"])
print("cycles: total %.3e | D stretches %.1f%% | D failed %.1f%% | D normal %.1f%% | rest (P, idle) %.1f%%" %
      (tot[0], 100 * tot[1] / tot[0], 100 * tot[2] / tot[0], 100 * tot[3] / tot[0],
       100 * (tot[0] - tot[1] - tot[2] - tot[3]) / tot[0]))
print("iterations %.3e (ff %.3e in %.3e stretches), transfers %.3e, req-its %.3e" %
      (tot[4], tot[5], tot[6], tot[7], s["n_request_iterations"].sum()))
