"""Measure the compressed FULL memory trace: bytes per iteration on whole C3 points (grid
corners of the hardware axes x 3 policies) and C1.  Writes profiles/r2/full_trace_codec.json.

    python tools/trace_codec_stats.py      (GPU)
"""
import json
import os
import sys
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import sweep_inputs as si  # noqa: E402
import paper_2503_08415_b200 as P  # noqa: E402

out = {"what": "compressed FULL memory trace (trace_codec.cuh): bytes of the stored stream per simulated iteration",
       "points": []}
base = si.c3()
cfg = replace(si.subset(base, hws=[0, 5, 1535, 1530, 767, 1000], policies=[0, 1, 2]),
              options=si.Options(trace_mode=si.FULL, trace_cap_bytes=6 << 20))
sw = P.Sweep(cfg)
sw.run()
s = sw.summaries()
for p in range(cfg.num_points):
    enc, n = sw.mem_trace_encoded(p)
    hw, pol, _, _ = cfg.point_coords(p)
    h = cfg.hws[hw]
    out["points"].append({"config": "C3", "peak_tflops": h.peak_flops / 1e12, "hbm_tbs": h.mem_bw / 1e12,
                          "capacity_gb": h.mem_capacity / 1e9, "policy": cfg.policies[pol].kind,
                          "iterations": int(n), "bytes": int(len(enc)), "bytes_per_iteration": len(enc) / max(1, n),
                          "overflow": bool(int(s["status_flags"][p]) & 1)})
c1 = replace(si.c1(), options=si.Options(trace_mode=si.FULL))
sw1 = P.Sweep(c1)
sw1.run()
enc, n = sw1.mem_trace_encoded(0)
out["points"].append({"config": "C1", "iterations": int(n), "bytes": int(len(enc)), "bytes_per_iteration": len(enc) / n})
bpi = [x["bytes_per_iteration"] for x in out["points"]]
out["bytes_per_iteration"] = {"min": min(bpi), "max": max(bpi), "mean_weighted": sum(x["bytes"] for x in out["points"]) /
                              sum(x["iterations"] for x in out["points"])}
out["raw_sample_bytes"] = 32
path = os.path.join(ROOT, "profiles", "r2", "full_trace_codec.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out["bytes_per_iteration"]))
