"""Small CUDA-path workload for compute-sanitizer (racecheck / synccheck / memcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [--variant helper|compact|full|pd]

Runs adversarial micro configurations (tiny KV pools, preemption storms, identical arrivals,
o = 1, STATIC / CONT / CONT_RATIO, SWAP / RECOMPUTE, FULL and BINNED traces) through the
C ABI on cuda:0 in the chosen kernel variant, and checks the per-point status flags (no
oracle: the sanitizer is the check).  The helper variant exercises the one-warp-per-SM kernel
whose helper warp consumes the simulating warp's rings through volatile shared-memory counters.
"""
import argparse
import os
import sys
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import sweep_inputs as si  # noqa: E402


def micro(rng, n_max=40):
    from test_gpu_parity import _micro
    return _micro(rng)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="helper", choices=["helper", "compact", "full", "pd"])
    ap.add_argument("--n", type=int, default=6)
    a = ap.parse_args()
    os.environ["TOKENSIM_HELPER"] = "1" if a.variant == "helper" else "0"
    import torch
    import paper_2503_08415_b200 as P
    rng = np.random.default_rng(99)
    bad = 0
    for i in range(a.n):
        cfg = micro(rng)
        if a.variant == "full":
            cfg = replace(cfg, policies=[replace(cfg.policies[0], iteration_mode=si.PREFILL_FIRST)])
        if a.variant == "pd":
            from test_gpu_parity import _micro_pd
            cfg = _micro_pd(rng)
        # a few identical points (TRACE mode: repeat the profile) so the compact variant runs
        # several warps per CTA
        cfg = replace(cfg, hws=list(cfg.hws) * 4)
        sw = P.Sweep(cfg)
        sw.run()
        torch.cuda.synchronize()
        s = sw.summaries()
        info = sw.run_info()
        err = int((s["status_flags"] & 16).sum())
        bad += err
        print(f"config {i}: points {len(s)} helper {info['helper_mode']} grid {info['sim_blocks']}x"
              f"{info['sim_warps_per_block']} internal-error flags {err}", flush=True)
        sw.close()
    print("sanitize_run done, internal errors:", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
