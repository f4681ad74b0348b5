import sys
from dataclasses import replace
import numpy as np
sys.path.insert(0, "tests")
import sweep_inputs as si
from test_gpu_parity import _micro_pd
from paper_2503_08415_b200 import api
from oracle import oracle as O

rng = np.random.default_rng(41)
fails = {}
for it in range(40):
    cfg = _micro_pd(rng)
    x = int(rng.integers(1, 5)); y = int(rng.integers(1, 9 - x))
    d0 = str(rng.choice([si.ROUND_ROBIN, si.LEAST_OUTSTANDING, si.LEAST_MEMORY]))
    for d in (si.ROUND_ROBIN, si.LEAST_OUTSTANDING, si.LEAST_MEMORY):
        for ff in (True, False):
            c2 = replace(cfg, options=replace(cfg.options, pd_prefill=x, pd_decode=y, dispatch=d, fast_forward=ff))
            sw = api.Sweep(c2); sw.run()
            bad = 0
            for p in range(c2.num_points):
                o = O.simulate(c2, p, want=("summary", "records"))
                if sw.records(p)["e2e_ns"].tolist() != o["records"]["e2e_ns"].tolist():
                    bad += 1
            key = (d, ff, c2.policies[0].kind)
            fails.setdefault(key, [0, 0])
            fails[key][0] += bad > 0
            fails[key][1] += 1
for k, v in sorted(fails.items()):
    print(k, "fail", v[0], "of", v[1])
