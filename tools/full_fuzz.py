"""Randomised check of the full kernel with (variant 6) and without (variant 1) the helper warp:
both must give the same bytes, and the helper run must equal the oracle.

    python tools/full_fuzz.py [--n 200] [--seed 11]

Configurations: the adversarial micro workloads of the parity tests under prefill-first or
chunked iterations (and the preload link for SWAP), plus small multi-round conversation sweeps
with and without the memory cache.  Prints one line per mismatch and a final count.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--seed", type=int, default=11)
    a = ap.parse_args()
    import paper_2503_08415_b200 as P
    from test_gpu_parity import _micro, check_points
    rng = np.random.default_rng(a.seed)
    bad = 0
    for it in range(a.n):
        if it % 4 == 3:  # multi-round conversations (generated workload)
            cfg = replace(si.c7(), workload=replace(si.c7().workload, num_requests=int(rng.integers(20, 200)),
                                                    rates=[float(rng.choice([0.5, 2.0, 8.0]))], seeds=[int(it)],
                                                    think_mean_s=float(rng.choice([0.5, 5.0]))),
                          policies=[si.Policy(preempt=str(rng.choice([si.SWAP, si.RECOMPUTE])))],
                          options=replace(si.c7().options, memory_cache=bool(rng.random() < 0.7),
                                          iteration_trace_cap=1 << 16, trace_mode=si.BINNED))
        else:
            cfg = _micro(rng)
            pol = cfg.policies[0]
            mode = str(rng.choice([si.PREFILL_FIRST, si.CHUNKED]))
            pol = replace(pol, iteration_mode=mode,
                          max_batched_tokens=int(rng.choice([max(pol.max_num_seqs, 16), 300])) if mode == si.CHUNKED
                          else pol.max_batched_tokens)
            opts = cfg.options
            if pol.preempt == si.SWAP and rng.random() < 0.4:
                opts = replace(opts, link_mode=si.PRELOAD, preload_buffer_bytes=int(rng.choice([1 << 14, 1 << 20, 1 << 34])))
            cfg = replace(cfg, policies=[pol], options=opts)
        outs = {}
        for v in ("1", "0"):
            os.environ["TOKENSIM_HELPER"] = v
            sw = P.Sweep(cfg)
            sw.run()
            info = sw.run_info()
            outs[v] = (sw, info["helper_mode"])
        os.environ.pop("TOKENSIM_HELPER", None)
        (h, hm), (p, pm) = outs["1"], outs["0"]
        msg = None
        if hm == 0 or pm != 0:
            msg = f"helper modes {hm} / {pm}"
        elif h.summaries().tobytes() != p.summaries().tobytes():
            msg = "summaries differ"
        else:
            for q in range(cfg.num_points):
                if (h.records(q).tobytes() != p.records(q).tobytes() or
                        h.iteration_trace(q).tobytes() != p.iteration_trace(q).tobytes() or
                        h.mem_trace(q).tobytes() != p.mem_trace(q).tobytes()):
                    msg = f"point {q} differs"
                    break
        if msg is None:
            try:
                check_points(h, cfg, list(range(cfg.num_points)), records=True, trace=True, iters=True)
            except AssertionError as e:
                msg = "oracle: " + str(e).splitlines()[0]
        if msg:
            bad += 1
            print(f"config {it}: {cfg.name} {cfg.policies[0].iteration_mode} {cfg.options.link_mode}: {msg}", flush=True)
        h.close()
        p.close()
    print(f"full_fuzz: {a.n} configurations, {bad} mismatching")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
