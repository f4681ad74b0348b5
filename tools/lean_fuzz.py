"""Randomised check of the lean unified kernels: 8 independent warps per SM (variant 4), the
helper-warp kernel with (variant 0) and without (variant 5) extended stretches -- all three must
give the same bytes, and equal the oracle.

    python tools/lean_fuzz.py [--n 200] [--seed 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--seed", type=int, default=5)
    a = ap.parse_args()
    import paper_2503_08415_b200 as P
    from test_gpu_parity import _micro, check_points
    rng = np.random.default_rng(a.seed)
    bad = 0
    for it in range(a.n):
        cfg = _micro(rng)
        outs = {}
        for name, env in (("v4", {"TOKENSIM_HELPER": "0"}), ("v0", {"TOKENSIM_HELPER": "1", "TOKENSIM_XS": "1"}),
                          ("v5", {"TOKENSIM_HELPER": "1", "TOKENSIM_XS": "0"})):
            for k in ("TOKENSIM_HELPER", "TOKENSIM_XS"):
                os.environ.pop(k, None)
            os.environ.update(env)
            sw = P.Sweep(cfg)
            sw.run()
            outs[name] = sw
        for k in ("TOKENSIM_HELPER", "TOKENSIM_XS"):
            os.environ.pop(k, None)
        ref = outs["v0"]
        msg = None
        for name, sw in outs.items():
            if sw.summaries().tobytes() != ref.summaries().tobytes():
                msg = f"{name} summaries differ"
                break
            for q in range(cfg.num_points):
                if (sw.records(q).tobytes() != ref.records(q).tobytes() or
                        sw.iteration_trace(q).tobytes() != ref.iteration_trace(q).tobytes() or
                        sw.mem_trace(q).tobytes() != ref.mem_trace(q).tobytes()):
                    msg = f"{name} point {q} differs"
                    break
            if msg:
                break
        if msg is None:
            try:
                check_points(ref, cfg, list(range(cfg.num_points)), records=True, trace=True, iters=True)
            except AssertionError as e:
                msg = "oracle: " + str(e).splitlines()[0]
        if msg:
            bad += 1
            print(f"config {it}: {msg}", flush=True)
        for sw in outs.values():
            sw.close()
    print(f"lean_fuzz: {a.n} configurations, {bad} mismatching")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
