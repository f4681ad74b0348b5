"""Minimal driver for ncu captures: one sweep run of a preset on cuda:0.

    python tools/prof_run.py --config c2 [--reps 1]
"""
import argparse
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
import torch  # noqa: E402

import sweep_inputs as si  # noqa: E402
import paper_2503_08415_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--points", type=int, default=0, help="run only the first N points")
ap.add_argument("--dump", default="", help="save per-point iterations / cycles / profile to this .npz")
ap.add_argument("--only", type=int, default=-1, help="run this one point alone (one warp on one SM)")
a = ap.parse_args()
cfg = si.PRESETS[a.config]()
sw = P.Sweep(cfg)
end = a.points or sw.num_points
beg = 0
if a.only >= 0:
    beg, end = a.only, a.only + 1
for _ in range(a.reps):
    sw.run(beg, end, 1)
    torch.cuda.synchronize()
    info = sw.run_info()
    s = sw.summaries()
    print(a.config, "points", len(s), "req-its", int(s["n_request_iterations"].sum()),
          "iters max", int(s["n_iterations"].max()), "sim ms %.3f" % info["ms_sim"],
          "grid", info["sim_blocks"], "x", info["sim_warps_per_block"], "smem/warp", info["smem_per_warp"])
if os.environ.get("PROFILE_POINTS"):
    import numpy as np
    prof = [sw.point_profile(p) for p in range(beg, end)]
    it = np.array([x["n_iterations"] for x in prof], dtype=np.float64)
    ff = np.array([x["ff_iterations"] for x in prof], dtype=np.float64)
    st = np.array([x["ff_stretches"] for x in prof], dtype=np.float64)
    cy = np.array([x["sm_cycles"] for x in prof], dtype=np.float64)
    ri = s["n_request_iterations"].astype(np.float64)
    normal = it - ff
    print("points", end, "sum cycles %.3e max %.3e" % (cy.sum(), cy.max()),
          "ff frac %.3f" % (ff.sum() / it.sum()), "avg stretch %.1f" % (ff.sum() / max(1, st.sum())))
    # least-squares split of cycles into per-normal-iteration, per-stretch and per-request-iteration costs
    X = np.stack([normal, st, ri], 1)
    coef, *_ = np.linalg.lstsq(X, cy, rcond=None)
    print("cycles ~ %.0f/normal-iter + %.0f/stretch + %.2f/req-iter" % tuple(coef))
    if a.dump:
        np.savez(a.dump, iters=it, ff=ff, stretches=st, cycles=cy, ri=ri,
                 cycles_ff=np.array([x["cycles_ff"] for x in prof], dtype=np.float64),
                 cycles_normal=np.array([x["cycles_normal"] for x in prof], dtype=np.float64),
                 cycles_ff_failed=np.array([x["cycles_ff_failed"] for x in prof], dtype=np.float64),
                 stretch_phase=np.array([x["stretch_phase_cycles"] for x in prof], dtype=np.float64),
                 normal_phase=np.array([x["normal_phase_cycles"] for x in prof], dtype=np.float64),
                 ff_cut=np.array([x["ff_cut"] for x in prof], dtype=np.float64),
                 preempt=s["n_preemptions"].astype(np.float64), sim_ms=info["ms_sim"])
    cuts = np.array([x["ff_cut"] for x in prof], dtype=np.float64).sum(0)
    print("all points: stretches ended by (memory / finish / arrival / head / 32+other):", cuts.astype(int).tolist())
    if os.environ.get("PROFILE_GROUPS"):  # worst point of each group of G consecutive points
        G = int(os.environ["PROFILE_GROUPS"])
        order = [g * G + int(np.argmax(cy[g * G:(g + 1) * G])) for g in range((end + G - 1) // G)]
    else:
        order = np.argsort(-cy)[:6]
    for p in order:
        x = prof[p]
        if a.only >= 0:
            print("  (point", a.only, "alone)")
        nn = max(1, x["n_iterations"] - x["ff_iterations"])
        print("  point", p, "cycles %.3e" % cy[p], "iters", int(it[p]), "ff", int(ff[p]), "stretches", int(st[p]),
              "req-its", int(ri[p]), "preempt", int(s["n_preemptions"][p]),
              "| cyc/stretch %.0f  cyc/normal %.0f  failed-ff %.2e" % (x["cycles_ff"] / max(1, x["ff_stretches"]),
                                                                       x["cycles_normal"] / nn, x["cycles_ff_failed"]))
        ns = max(1, x["ff_stretches"])
        print("     stretch phases (cycles/stretch):", " ".join("%.0f" % (c / ns) for c in x["stretch_phase_cycles"]))
        print("     normal phases (cycles/iter):", " ".join("%.0f" % (c / nn) for c in x["normal_phase_cycles"]))
        print("     failed FF attempts (not quiet / memory / arrival / head / other):", x["ff_failed"])
        print("     stretches ended by (memory / finish / arrival / head / 32+other):", x["ff_cut"])
