"""Randomised parity sweep of the xP:yD node kernel against the oracle's sequential node loop
(a longer run of tests/test_gpu_parity.py::test_node_epoch_stress's generator).

    python tools/node_fuzz.py [--n 300] [--seed 7] [--pair] [--horizon]

Every configuration: random x:y (x + y <= 8), dispatch policy, arrivals (sparse, dense, bursts of
equal times), lengths, KV pool, block size, preemption mode, trace mode, fast-forward; all points
compared byte for byte (summaries, records, every worker's trace, iteration records by
(worker, k)).  --pair: 1P:1D pairs through the pair kernel, which must also give the bytes of the
same pairs run through the node kernel (options.node_loop).  Prints one line per mismatch and a
final count.
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
    ap.add_argument("--n", type=int, default=300)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--pair", action="store_true")
    ap.add_argument("--horizon", action="store_true", help="stop every point at a random horizon")
    a = ap.parse_args()
    import paper_2503_08415_b200 as P
    from test_gpu_parity import _micro_pd, check_pd_points
    rng = np.random.default_rng(a.seed)
    bad = 0
    for it in range(a.n):
        cfg = _micro_pd(rng)
        n = int(rng.integers(5, 200))
        base = np.sort(rng.integers(0, int(rng.choice([5e7, 2e8, 2e9, 2e10])), n))
        if it % 3 == 0:
            base = np.sort(np.repeat(base[: max(1, n // int(rng.integers(2, 6)))], 6)[:n])
        p = rng.integers(1, 64, len(base))
        o = rng.integers(1, 64, len(base))
        w = replace(cfg.workload, num_requests=len(base), trace_arrival_ns=base.tolist(), trace_prompt=p.tolist(),
                    trace_output=o.tolist())
        x = 1 if a.pair else int(rng.integers(1, 5))
        y = 1 if a.pair else int(rng.integers(1, 9 - x))
        d = str(rng.choice([si.ROUND_ROBIN, si.LEAST_OUTSTANDING, si.LEAST_MEMORY]))
        cfg = replace(cfg, workload=w, options=replace(cfg.options, pd_prefill=x, pd_decode=y, dispatch=d))
        if a.horizon:  # somewhere inside the arrival span, or a little past it
            hz = int(rng.integers(1, int(base[-1]) + 2)) + int(rng.choice([0, 0, 10 ** 8]))
            cfg = replace(cfg, options=replace(cfg.options, horizon_ns=hz))
        sw = P.Sweep(cfg)
        sw.run()
        try:
            check_pd_points(sw, cfg, list(range(cfg.num_points)), iters=True)
            if a.pair:
                nl = P.Sweep(replace(cfg, options=replace(cfg.options, node_loop=True)))
                nl.run()
                assert nl.summaries().tobytes() == sw.summaries().tobytes(), "node loop summaries differ"
                for q in range(cfg.num_points):
                    assert nl.records(q).tobytes() == sw.records(q).tobytes(), f"node loop records differ ({q})"
                nl.close()
        except AssertionError as e:
            bad += 1
            print(f"config {it}: x={x} y={y} {d} n={len(base)}: {str(e).splitlines()[0]}", flush=True)
        sw.close()
    print(f"node_fuzz{' --pair' if a.pair else ''}{' --horizon' if a.horizon else ''}: {a.n} configurations, {bad} mismatching")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
