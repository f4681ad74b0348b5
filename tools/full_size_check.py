"""Larger samples of the full-size bench configurations against the oracle (the test suite checks
16 / 12 / 8 points of C3 / C4 / C5): every k-th point of the sweep exactly as bench.py runs it,
summaries and per-request records byte for byte.

    python tools/full_size_check.py [--c3 16] [--c4 12] [--c5 32] [--c6 4] [--c2 k] [--c7 k] [--c8 k] [--c9 k]
    (every k-th point; 0 skips a config)
"""
import argparse
import os
import sys
import time
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import sweep_inputs as si  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3", type=int, default=16)
    ap.add_argument("--c4", type=int, default=12)
    ap.add_argument("--c5", type=int, default=32)
    ap.add_argument("--c6", type=int, default=4)
    ap.add_argument("--c2", type=int, default=0)
    ap.add_argument("--c7", type=int, default=0)
    ap.add_argument("--c8", type=int, default=0)
    ap.add_argument("--c9", type=int, default=0)
    a = ap.parse_args()
    import paper_2503_08415_b200 as P
    from test_gpu_parity import check_points, check_pd_points
    total_bad = 0
    c5 = replace(si.c5(), workload=replace(si.c5().workload, seeds=[0]))  # bench.py's per-GPU share
    for name, cfg, every, pd in (("c3", si.c3(), a.c3, False), ("c4", si.c4(), a.c4, False),
                                 ("c5 (8,192 pairs)", c5, a.c5, True), ("c6", si.c6(), a.c6, True),
                                 ("c2", si.c2(), a.c2, False), ("c7", si.c7(), a.c7, False),
                                 ("c8", si.c8(), a.c8, False), ("c9", si.c9(), a.c9, False)):
        if every <= 0:
            continue
        t0 = time.time()
        sw = P.Sweep(cfg)
        sw.run()
        pts = list(range(0, cfg.num_points, every))
        try:
            if pd:
                check_pd_points(sw, cfg, pts)
            else:
                check_points(sw, cfg, pts, records=True)
            res = "equal"
        except AssertionError as e:
            total_bad += 1
            res = "MISMATCH " + str(e).splitlines()[0]
        print(f"{name}: {len(pts)} of {cfg.num_points} points (every {every}th) vs the oracle: {res} "
              f"({time.time() - t0:.0f} s)", flush=True)
        sw.close()
    return 1 if total_bad else 0


if __name__ == "__main__":
    sys.exit(main())
