"""A/B timing of library builds: each listed library runs the same presets in its own process.

    python tools/ab.py LIB_A LIB_B [--configs c2,c3s4,c4s4] [--reps 3]

Prints best-of-reps sim-kernel ms per (library, config) and a hash of every summary, record and
iteration-trace byte, so a faster build is also shown to be bit-identical.  c3s / c4s are
subsets (every k-th point: c3s4 = every 4th point of C3).
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, json, os, sys
sys.path.insert(0, %(root)r)
import numpy as np, torch
import sweep_inputs as si
import paper_2503_08415_b200 as P
res = {}
for name in %(configs)r:
    base, _, st = name.partition("s")
    cfg = si.PRESETS[base]()
    sw = P.Sweep(cfg)
    npts = sw.num_points
    stride = int(st) if st else 1
    best = best_s = 1e30
    for _ in range(%(reps)d):
        sw.run(0, npts, stride)
        torch.cuda.synchronize()
        ri = sw.run_info()
        best = min(best, ri["ms_sim"])
        best_s = min(best_s, ri["ms_summary"])
    s = sw.summaries()
    h = hashlib.sha256(np.ascontiguousarray(s).tobytes())
    for q in range(0, len(s), max(1, len(s) // 16)):
        h.update(np.ascontiguousarray(sw.records(q * stride)).tobytes())
    res[name] = {"ms_sim": best, "ms_summary": best_s, "points": int(len(s)), "req_its": int(s["n_request_iterations"].sum()),
                 "hash": h.hexdigest()[:16]}
print("RESULT " + json.dumps(res))
"""


def main():
    args = sys.argv[1:]
    configs = ["c2", "c3s4", "c4s4"]
    reps = 3
    if "--configs" in args:
        i = args.index("--configs")
        configs = args[i + 1].split(",")
        del args[i:i + 2]
    if "--reps" in args:
        i = args.index("--reps")
        reps = int(args[i + 1])
        del args[i:i + 2]
    out = {}
    for lib in args:
        env = dict(os.environ, TOKENSIM_LIB=os.path.abspath(lib))
        code = CHILD % {"root": ROOT, "configs": configs, "reps": reps}
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        if r.returncode or not line:
            print(lib, "FAILED", r.returncode, r.stderr[-2000:])
            continue
        out[lib] = json.loads(line[0][7:])
        for c, v in out[lib].items():
            print("%-40s %-4s %9.3f ms  %.3e req-it/s  summary %8.3f ms  hash %s" %
                  (os.path.basename(lib), c, v["ms_sim"], v["req_its"] / v["ms_sim"] * 1e3, v["ms_summary"], v["hash"]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
