"""Debug helper: first node micro config that diverges from the oracle; prints details."""
import sys
from dataclasses import replace
import numpy as np
sys.path.insert(0, "tests")
import sweep_inputs as si
from test_gpu_parity import _micro_pd
from paper_2503_08415_b200 import api
from oracle import oracle as O

rng = np.random.default_rng(41)
for it in range(40):
    cfg = _micro_pd(rng)
    x = int(rng.integers(1, 5)); y = int(rng.integers(1, 9 - x))
    d = str(rng.choice([si.ROUND_ROBIN, si.LEAST_OUTSTANDING, si.LEAST_MEMORY]))
    cfg = replace(cfg, options=replace(cfg.options, pd_prefill=x, pd_decode=y, dispatch=d))
    for ff in (True, False):
        c2 = replace(cfg, options=replace(cfg.options, fast_forward=ff))
        sw = api.Sweep(c2); sw.run()
        for p in range(c2.num_points):
            o = O.simulate(c2, p, want=("summary", "records", "iters"))
            g = sw.iteration_trace(p)
            gi = g[np.lexsort((g["k"], g["worker"]))]
            oi = o["iters"][np.lexsort((o["iters"]["k"], o["iters"]["worker"]))]
            ok = len(gi) == len(oi)
            first = None
            for i in range(min(len(gi), len(oi))):
                a = (int(gi["worker"][i]), int(gi["k"][i]), int(gi["t_start_ns"][i]), int(gi["T_ns"][i]), int(gi["n_prefill"][i]), int(gi["n_decode"][i]), int(gi["n_admitted"][i]), int(gi["n_finished"][i]), int(gi["blocks_in_use"][i]))
                b = (int(oi["worker"][i]), int(oi["k"][i]), int(oi["t_start"][i]), int(oi["T_ns"][i]), int(oi["S_p"][i]), int(oi["D"][i]), int(oi["n_admitted"][i]), int(oi["n_finished"][i]), int(oi["blocks"][i]))
                if a != b:
                    first = i; break
            if first is not None or not ok:
                print("case", it, "x,y,d", x, y, d, "ff", ff, "point", p, "pol", c2.policies[0], "link", c2.options.pd_link_bw,
                      "hws", [(h.kv_blocks_override, h.peak_flops, h.mem_bw) for h in c2.hws], "n", c2.workload.num_requests)
                i0 = max(0, (first or 0) - 3)
                for i in range(i0, min(i0 + 8, len(gi), len(oi))):
                    print(" gpu", i, tuple(int(gi[f][i]) for f in ("worker","k","t_start_ns","T_ns","n_prefill","n_decode","n_admitted","n_finished","blocks_in_use")))
                    print(" ora", i, tuple(int(oi[f][i]) for f in ("worker","k","t_start","T_ns","S_p","D","n_admitted","n_finished","blocks")))
                print("gpu nit", len(gi), "ora nit", len(oi))
                w = list(zip(c2.workload.trace_arrival_ns, c2.workload.trace_prompt, c2.workload.trace_output))
                print("reqs", w[:60])
                sys.exit(0)
print("all ok")
