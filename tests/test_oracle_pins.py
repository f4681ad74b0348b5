"""Pins for the CPU oracle (-m "not gpu").

Each test ties the oracle to something other than itself: known-answer vectors
(Random123), published model facts (parameter counts), closed forms
(roofline limits, Lindley recursion, isolated requests), hand-worked traces
(SURVEY §8(c.8)), statistics the paper/spec fixes (Poisson arrivals S:111/S:125)
and invariants.  Golden values live in
tests/golden/*.json with their citations.
"""
import json
import math
import os
from dataclasses import replace

import numpy as np
import pytest

import sweep_inputs as si

GOLD = os.path.join(os.path.dirname(__file__), "golden")
LN2 = float.fromhex("0x1.62e42fefa39efp-1")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def trace_cfg(reqs, hw=si.A100_IDEAL, pol=si.Policy(), model=si.LLAMA2_7B, **opt):
    w = si.Workload(len(reqs), [1.0], [0], len_dist=si.TRACE,
                    trace_arrival_ns=[r[0] for r in reqs], trace_prompt=[r[1] for r in reqs],
                    trace_output=[r[2] for r in reqs], prompt_table=None, output_table=None)
    return si.SweepConfig("trace", model, [hw], [pol], w, si.Options(**opt))


# ------------------------------------------------------------------ a.1 generator
def test_philox_known_answers(oracle_lib):
    for v in gold("philox_kat.json")["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        assert list(oracle_lib.philox(ctr, key)) == [int(x, 16) for x in v["out"]]


def test_det_log_exact_cases(oracle_lib):
    assert oracle_lib.det_log(1.0) == 0.0
    for k in range(1, 64):
        assert oracle_lib.det_log(2.0 ** -k) == (-k) * LN2


def test_det_log_matches_libm(oracle_lib):
    rng = np.random.default_rng(1)
    us = np.concatenate([rng.random(20000), 1.0 - rng.random(2000) * 1e-12,
                         np.exp(-rng.random(2000) * 700)])
    worst_ulp = 0.0
    for u in us:
        if u <= 0.0:
            continue
        ref = math.log(u)
        got = oracle_lib.det_log(float(u))
        if ref != 0.0:
            worst_ulp = max(worst_ulp, abs(got - ref) / math.ulp(ref))
    # within 2 ulp of libm log (SURVEY c.8 quotes <= 3.6e-16 relative on its sample)
    assert worst_ulp <= 2.0, worst_ulp


def _gen(cfg):
    from oracle import oracle as O
    return O.workload(cfg, 0)


def test_arrivals_are_poisson(oracle_lib):
    from scipy import stats
    lam = 2.0
    cfg = si.SweepConfig("w", si.LLAMA2_7B, [si.A100], [si.Policy()], si.Workload(50000, [lam], [7]))
    a, p, o = _gen(cfg)
    gaps = np.diff(np.concatenate([[0], a])) / 1e9
    assert gaps.min() >= 0
    # mean inter-arrival within [0.45, 0.55] s at qps = 2 (we use a 3% band)
    assert abs(gaps.mean() - 1 / lam) < 0.03 / lam
    # exponential shape (no dropped minus sign, no wrong scale)
    assert stats.kstest(gaps, "expon", args=(0, 1 / lam)).pvalue > 1e-3
    # counts in disjoint equal windows have dispersion index in [0.8, 1.2]
    a1 = a[:10000] / 1e9
    counts = np.bincount(np.floor(a1).astype(int))[:-1]
    assert 0.8 <= counts.var() / counts.mean() <= 1.2


def test_workload_determinism_and_seeds(oracle_lib):
    cfg = si.SweepConfig("w", si.LLAMA2_7B, [si.A100], [si.Policy()], si.Workload(1000, [2.0], [7, 8]))
    from oracle import oracle as O
    a0, p0, o0 = O.workload(cfg, 0)
    a1, p1, o1 = O.workload(cfg, 0)
    b, q, r = O.workload(cfg, 1)
    assert (a0 == a1).all() and (p0 == p1).all() and (o0 == o1).all()
    assert not (a0 == b).all() and not (p0 == q).all()
    # rate only rescales the exponentials: a(lambda=4) ~= a(lambda=2)/2
    cfg4 = replace(cfg, workload=replace(cfg.workload, rates=[4.0]))
    a4, p4, o4 = O.workload(cfg4, 0)
    assert (p4 == p0).all() and (o4 == o0).all()
    assert np.abs(a4 - a0 / 2).max() <= 1000  # one rounding per gap, <= n * 1 ns


def test_length_table_statistics(oracle_lib):
    n = 200000
    cfg = si.SweepConfig("w", si.LLAMA2_7B, [si.A100], [si.Policy()], si.Workload(n, [1.0], [7]))
    a, p, o = _gen(cfg)
    for vals, t in ((p, si.SHAREGPT_PROMPT), (None, si.SHAREGPT_OUTPUT)):
        edges = list(t.thr) + [2 ** 32]
        probs = np.diff([0] + edges) / 2 ** 32
        if vals is None:
            # unclamped output draws: only requests whose clamp is inactive
            mask = o < 2048 - p
            vals = o[mask]
            probs_eff = None
        else:
            probs_eff = probs
        bucket = np.searchsorted(np.asarray(t.hi), vals, side="right")
        assert (vals >= t.lo[0]).all() and (vals < t.hi[-1]).all()
        if probs_eff is not None:
            freq = np.bincount(bucket, minlength=len(t.lo)) / len(vals)
            sig = np.sqrt(probs_eff * (1 - probs_eff) / len(vals))
            assert (np.abs(freq - probs_eff) < 5 * sig + 1e-12).all(), (freq, probs_eff)
            # analytic mean of lo + floor(y*(hi-lo)/2^32) with y uniform
            mean = sum(pr * (lo + (hi - lo - 1) / 2) for pr, lo, hi in zip(probs, t.lo, t.hi))
            assert abs(vals.mean() - mean) / mean < 0.01
            # within-bucket uniformity of the multiply-shift draw (bucket [64,128))
            sel = vals[bucket == 3]
            assert abs(sel.mean() - (64 + 127) / 2) < 1.0
    assert (p + o <= 2048).all() and (o >= 1).all()
    assert abs(p.mean() - 161.31) < 2.0  # vLLM's published ShareGPT prompt mean (A25, ext)


def test_fixed_and_uniform_lengths(oracle_lib):
    w = si.Workload(5000, [1.0], [3], len_dist=si.FIXED, prompt_a=128, output_a=1024)
    a, p, o = _gen(si.SweepConfig("w", si.LLAMA2_7B, [si.A100], [si.Policy()], w))
    assert (p == 128).all() and (o == 1024).all()
    w = si.Workload(20000, [1.0], [3], len_dist=si.UNIFORM, prompt_a=10, prompt_b=20, output_a=1, output_b=4)
    a, p, o = _gen(si.SweepConfig("w", si.LLAMA2_7B, [si.A100], [si.Policy()], w))
    assert p.min() == 10 and p.max() == 20 and o.min() == 1 and o.max() == 4
    cnt = np.bincount(o)[1:]
    assert (np.abs(cnt / cnt.sum() - 0.25) < 0.02).all()


# ------------------------------------------------------------------ c.1 constants
BIG = si.Hw(mem_capacity=10 ** 12)


def _one(model, hw=None, pol=si.Policy()):
    if hw is None:
        hw = BIG if model is si.LLAMA2_70B else si.A100
    return si.SweepConfig("m", model, [hw], [pol], si.Workload(1, [1.0], [0]))


def test_weight_bytes_match_published_params(oracle_lib):
    pub = gold("llama2_published.json")["models"]
    for m in (si.LLAMA2_7B, si.LLAMA2_13B, si.LLAMA2_70B):
        d = oracle_lib.derive(_one(m))
        ref = pub[m.name]
        assert (m.num_layers, m.hidden, m.num_heads, m.num_kv_heads) == (ref["L"], ref["h"], ref["n_heads"], ref["n_kv"])
        assert d["W"] == 2 * ref["params"]
        assert d["kvb"] == ref["kvb"]
        assert d["block_bytes"] == 16 * ref["kvb"]


def test_block_capacity_ladder(oracle_lib):
    got = [oracle_lib.derive(_one(si.LLAMA2_7B, si.Hw(mem_capacity=c * 10 ** 9)))["total_blocks"]
           for c in (20, 40, 80, 160, 320, 640)]
    assert got == [658, 2923, 7453, 16513, 34633, 70872]
    assert oracle_lib.derive(_one(si.LLAMA2_13B))["total_blocks"] == 3812
    assert [oracle_lib.derive(_one(si.LLAMA2_70B, h))["total_blocks"] for h in si.c4_hws()] == [2679, 31670, 89654]
    # capacity below the weights is rejected ("lower than the model parameter size")
    with pytest.raises(Exception):
        oracle_lib.derive(_one(si.LLAMA2_7B, si.Hw(mem_capacity=10 * 10 ** 9)))


def test_ratio_limit(oracle_lib):
    d = oracle_lib.derive(_one(si.LLAMA2_7B, pol=si.Policy(kind=si.CONT_RATIO, max_mem_ratio=0.9)))
    assert d["ratio_limit"] == math.floor(0.9 * 7453)


# ------------------------------------------------------------------ a.6 cost model
def _t(cfg, prefills=(), decodes=(), swap=0):
    from oracle import oracle as O
    return O.iter_time_ns(cfg, [(P, 0) for P in prefills], decodes, swap)


def test_cost_closed_form_rows(oracle_lib):
    for row in gold("cost_closed_form.json")["rows"]:
        hw = si.A100 if row.get("defaults") else si.A100_IDEAL
        cfg = _one(si.LLAMA2_7B, hw)
        dec = [c for c, b in row["decodes"] for _ in range(b)]
        assert _t(cfg, row["prefills"], dec) == row["T_ns"], row["desc"]


@pytest.mark.parametrize("model", [si.LLAMA2_7B, si.LLAMA2_13B, si.LLAMA2_70B])
def test_cost_memory_bound_limit(oracle_lib, model):
    """Infinite FLOP/s: a decode step reads every linear weight once plus the KV
    of its context; per extra context token exactly kvb bytes."""
    pub = gold("llama2_published.json")["models"][model.name]
    B = 2.039e12
    cfg = _one(model, si.Hw(peak_flops=1e30, mem_bw=B, eff_flops=1, eff_bw=1, iter_overhead_s=0,
                                    mem_capacity=10 ** 12))
    L, h, V = model.num_layers, model.hidden, model.vocab
    # weights the decode step touches = all params except the input embedding and the norms (A19)
    wbytes = 2 * (pub["params"] - V * h - (2 * L + 1) * h)
    # generous bound on activation + logit bytes per token (far below any weight matrix)
    act = L * 2 * 8 * (h + model.ffn_dim) + 4 * V
    t1 = _t(cfg, decodes=[1])
    assert 0 <= t1 * 1e-9 * B - wbytes < act
    t2 = _t(cfg, decodes=[1001])
    assert abs((t2 - t1) - 1000 * pub["kvb"] / B * 1e9) <= 2
    # batch: b decodes share one weight read
    tb = _t(cfg, decodes=[1] * 64)
    assert 0 <= tb * 1e-9 * B - wbytes < 64 * act


@pytest.mark.parametrize("model", [si.LLAMA2_7B, si.LLAMA2_70B])
def test_cost_compute_bound_limit(oracle_lib, model):
    """Infinite bandwidth: a prefill of P tokens costs 2 FLOPs per linear weight per token
    plus causal attention 4*q*L*P(P+1)/2 plus one LM-head row."""
    pub = gold("llama2_published.json")["models"][model.name]
    F = 312e12
    cfg = _one(model, si.Hw(peak_flops=F, mem_bw=1e30, eff_flops=1, eff_bw=1, iter_overhead_s=0,
                                    mem_capacity=10 ** 12))
    L, h, V = model.num_layers, model.hidden, model.vocab
    q = model.num_heads * model.head_dim
    linear = pub["params"] - 2 * V * h - (2 * L + 1) * h
    for P in (1, 128, 2048):
        flops = 2 * P * linear + 4 * q * L * P * (P + 1) // 2 + 2 * h * V
        assert abs(_t(cfg, prefills=[P]) - flops / F * 1e9) <= 2


def test_cost_tp_allreduce_and_swap_terms(oracle_lib):
    m = si.LLAMA2_70B
    base = si.Hw(peak_flops=2 * 312e12, mem_bw=2 * 2.039e12, mem_capacity=160 * 10 ** 9,
                 eff_flops=1, eff_bw=1, iter_overhead_s=0, host_link_bw=32e9)
    tp = replace(base, tp_degree=2, tp_link_bw=300e9)
    for N in (1, 37):
        t0 = _t(_one(m, base), decodes=[100] * N)
        t1 = _t(_one(m, tp), decodes=[100] * N)
        # ring all-reduce: 2(t-1)/t * N*h*s bytes per all-reduce, 2 per layer
        expect = 2 * m.num_layers * (2 * 1 / 2) * N * m.hidden * 2 / 300e9 * 1e9
        assert abs((t1 - t0) - expect) <= 2
    x = 7 * 16 * 327680
    assert abs(_t(_one(m, base), decodes=[5], swap=x) - _t(_one(m, base), decodes=[5]) - x / 32e9 * 1e9) <= 1


def test_cost_monotone_random_plans(oracle_lib):
    rng = np.random.default_rng(5)
    cfg = _one(si.LLAMA2_13B, si.A100)
    for _ in range(100):
        pf = list(rng.integers(1, 2048, rng.integers(0, 4)))
        dec = list(rng.integers(1, 2048, rng.integers(0, 40)))
        if not pf and not dec:
            dec = [1]
        t = _t(cfg, pf, dec)
        assert _t(cfg, pf, dec + [int(rng.integers(1, 2048))]) >= t
        assert _t(cfg, pf + [int(rng.integers(1, 2048))], dec) >= t
        if dec:
            assert _t(cfg, pf, [c + 1 for c in dec]) >= t
    # phase classes: prefill 2048 compute-bound, decode b=1 memory-bound
    fast_bw = si.Hw(mem_bw=2.039e14)
    fast_f = si.Hw(peak_flops=312e14)
    assert _t(_one(si.LLAMA2_7B, fast_f), prefills=[2048]) < 0.2 * _t(_one(si.LLAMA2_7B), prefills=[2048])
    assert _t(_one(si.LLAMA2_7B, fast_bw), decodes=[1]) < 0.2 * _t(_one(si.LLAMA2_7B), decodes=[1])
    assert abs(_t(_one(si.LLAMA2_7B, si.Hw(peak_flops=624e12)), decodes=[1])
               / _t(_one(si.LLAMA2_7B), decodes=[1]) - 1) < 0.01


def test_decode_stretch_times_nondecreasing(oracle_lib):
    """The kernel's fast-forward takes a stretch's largest token gap as its last iteration's T
    (DESIGN §8 A/B log): in a decode-only stretch only C_d grows (every context +1 per iteration),
    so T_j must be nondecreasing in j for every model, profile and TP degree, rounding included."""
    rng = np.random.default_rng(11)
    hws = [si.A100, si.A100_IDEAL, si.Hw(peak_flops=2.5e15, mem_bw=8e12)] + \
          [si.Hw(tp_degree=t, tp_link_bw=300e9) for t in (2, 4, 8)]
    for model in (si.LLAMA2_7B, si.LLAMA2_13B, si.LLAMA2_70B):
        for hw in hws:
            cfg = _one(model, hw)
            for _ in range(4):
                dec = [int(x) for x in rng.integers(1, 4096, int(rng.integers(1, 64)))]
                ts = [_t(cfg, decodes=[c + j for c in dec]) for j in range(32)]
                assert all(a <= b for a, b in zip(ts, ts[1:])), (model.name, hw, ts)


# ------------------------------------------------------------------ a.2-a.7 hand-worked traces
def _sim(cfg, **kw):
    from oracle import oracle as O
    return O.simulate(cfg, 0, check_invariants=True, **kw)


def test_single_request_trace(oracle_lib):
    g = gold("hand_traces.json")["single"]
    cfg = trace_cfg(g["requests"])
    assert _t(cfg, prefills=[20]) == g["T_pre_20"]
    assert _t(cfg, decodes=[21]) == g["T_dec_21"] and _t(cfg, decodes=[22]) == g["T_dec_22"]
    r = _sim(cfg, keep_events=True, want=("summary", "records", "iters", "events"))
    rec = r["records"][0]
    assert (rec["ttft_ns"], rec["e2e_ns"], rec["mtpot_ns"]) == (g["ttft"], g["e2e"], g["mtpot"])
    allocs = [int(e["block"]) for e in r["events"] if e["kind"] == 1]
    assert allocs == g["blocks"]
    s = r["summary"]
    assert s["n_iterations"] == 3 and s["n_request_iterations"] == 3
    assert abs(s["stat"][1][0] - (g["e2e"] - g["ttft"]) / 2 / 1e9) < 1e-18  # TPOT 6,488,846.5 ns


def test_two_request_trace(oracle_lib):
    g = gold("hand_traces.json")["two"]
    r = _sim(trace_cfg(g["requests"]), keep_events=True, want=("summary", "records", "iters", "events"))
    assert list(r["iters"]["T_ns"]) == g["iter_T"]
    assert list(r["iters"]["S_p"]) == [1, 1, 0] and list(r["iters"]["D"]) == [0, 1, 2]
    for i, key in ((0, "r0"), (1, "r1")):
        assert r["records"][i]["ttft_ns"] == g[key]["ttft"]
        assert r["records"][i]["e2e_ns"] == g[key]["e2e"]
    for rid, blocks in g["blocks"].items():
        got = [int(e["block"]) for e in r["events"] if e["kind"] == 1 and e["req"] == int(rid)]
        assert got == blocks


def test_isolated_requests_closed_form(oracle_lib):
    g = gold("hand_traces.json")["isolated"]
    cfg = trace_cfg([(0, g["p"], g["o"]), (10 ** 12, g["p"], g["o"])])
    r = _sim(cfg)
    expect_e2e = _t(cfg, prefills=[g["p"]]) + sum(_t(cfg, decodes=[g["p"] + j]) for j in range(1, g["o"]))
    for rec in r["records"]:
        assert rec["ttft_ns"] == g["ttft"] and rec["e2e_ns"] == g["e2e"] == expect_e2e


@pytest.mark.parametrize("mode", [si.SWAP, si.RECOMPUTE])
def test_preemption_hand_trace(oracle_lib, mode):
    g = gold("hand_traces.json")["preemption"]
    model = replace(si.LLAMA2_7B, max_model_len=g["max_model_len"])
    hw = replace(si.A100_IDEAL, kv_blocks_override=g["total_blocks"])
    pol = si.Policy(preempt=mode, block_size=g["block_size"])
    cfg = trace_cfg(g["requests"], hw=hw, pol=pol, model=model)
    r = _sim(cfg, keep_events=True, want=("summary", "records", "iters", "events"))
    s, it = r["summary"], r["iters"]
    assert s["n_iterations"] == g["iterations"] and s["n_request_iterations"] == g["request_iterations"]
    ev = [[int(e["k"]), int(e["kind"]), int(e["req"]), int(e["block"])] for e in r["events"]]
    assert ev == g["events"]
    assert list(it["m"]) == [0, 0, 0, 0, 0, 1, 0] and list(it["n_resumed"]) == [0] * 6 + [1]
    bb = g["block_size"] * 524288
    if mode == si.SWAP:
        assert s["swap_out_bytes"] == g["swap_blocks_out"] * bb and s["swap_in_bytes"] == g["swap_blocks_in"] * bb
        assert list(it["S_p"]) == [2, 0, 0, 0, 0, 0, 0]
        assert it["C_d"][6] == 9
    else:
        assert s["swap_out_bytes"] == 0 and s["swap_in_bytes"] == 0
        assert list(it["S_p"]) == [2, 0, 0, 0, 0, 0, 1] and it["N_p"][6] == 9
    r1 = r["records"][1]
    assert r1["n_preempt"] == 1 and r["records"][0]["n_preempt"] == 0
    assert r1["mtpot_ns"] == it["T_ns"][5] + it["T_ns"][6]           # gap spans It6 + It7
    assert r1["mtpot_ns"] > max(it["T_ns"][1:5])


def test_single_server_lindley(oracle_lib):
    """max_num_seqs = 1 is the FCFS single-server queue: start_i = max(a_i, fin_{i-1})."""
    rng = np.random.default_rng(11)
    n = 25
    a = np.cumsum(rng.integers(0, 400_000_000, n))
    p = rng.integers(1, 300, n)
    o = rng.integers(1, 40, n)
    cfg = trace_cfg(list(zip(a.tolist(), p.tolist(), o.tolist())), pol=si.Policy(max_num_seqs=1))
    r = _sim(cfg)
    fin = 0
    for i in range(n):
        start = max(int(a[i]), fin)
        tp = _t(cfg, prefills=[int(p[i])])
        td = [_t(cfg, decodes=[int(p[i]) + j]) for j in range(1, int(o[i]))]
        fin = start + tp + sum(td)
        rec = r["records"][i]
        assert rec["ttft_ns"] == start + tp - a[i]
        assert rec["e2e_ns"] == fin - a[i]
        assert rec["mtpot_ns"] == (max(td) if td else 0)


def test_static_batching_bubbles(oracle_lib):
    """outputs {2,3,5,8}, batch 4 -> the next batch starts only after the 8-token
    request finishes (P:426 'shorter requests have to wait'); continuous batching admits
    the fifth request as soon as a slot frees."""
    reqs = [(0, 10, 2), (0, 10, 3), (0, 10, 5), (0, 10, 8), (0, 10, 3)]
    st = _sim(trace_cfg(reqs, pol=si.Policy(kind=si.STATIC, max_num_seqs=4)))["records"]
    co = _sim(trace_cfg(reqs, pol=si.Policy(kind=si.CONT, max_num_seqs=4)))["records"]
    assert st[4]["ttft_ns"] > st[3]["e2e_ns"]
    assert co[4]["ttft_ns"] < co[3]["e2e_ns"]
    assert co["e2e_ns"].max() <= st["e2e_ns"].max()                        # S:361 makespan
    # batch of one degenerates to sequential FCFS
    b1s = _sim(trace_cfg(reqs, pol=si.Policy(kind=si.STATIC, max_num_seqs=1)))["records"]
    b1c = _sim(trace_cfg(reqs, pol=si.Policy(kind=si.CONT, max_num_seqs=1)))["records"]
    assert (b1s == b1c).all()


def test_mixed_arrival_joins_next_boundary(oracle_lib):
    """a request arriving mid-iteration joins at the next boundary."""
    cfg = trace_cfg([(0, 100, 50), (1, 100, 5)])
    r = _sim(cfg, want=("summary", "records", "iters"))
    it = r["iters"]
    assert it["S_p"][0] == 1 and it["S_p"][1] == 1 and it["D"][1] == 1
    assert r["records"][1]["ttft_ns"] == it["T_ns"][0] + it["T_ns"][1] - 1


# ------------------------------------------------------------------ invariants / properties
def _random_micro(rng):
    n = int(rng.integers(1, 60))
    a = np.sort(rng.integers(0, 3_000_000_000, n))
    p = rng.integers(1, 64, n)
    o = rng.integers(1, 64, n)
    mml = 128
    model = replace(si.LLAMA2_7B, max_model_len=mml)
    bs = int(rng.choice([1, 4, 16]))
    total = int(rng.integers(-(-mml // bs), -(-mml // bs) + 40))
    hw = replace(si.A100, kv_blocks_override=total)
    kind = rng.choice([si.STATIC, si.CONT, si.CONT_RATIO])
    pol = si.Policy(kind=str(kind), preempt=str(rng.choice([si.SWAP, si.RECOMPUTE])),
                    max_mem_ratio=float(rng.choice([0.3, 0.7, 1.0])),
                    max_num_seqs=int(rng.choice([1, 3, 8, 256])), block_size=bs,
                    max_batched_tokens=int(rng.choice([mml, 300, si.UINT32_MAX])),
                    watermark_blocks=int(rng.integers(0, total - (-(-mml // bs)) + 1)))
    return trace_cfg(list(zip(a.tolist(), p.tolist(), o.tolist())), hw=hw, pol=pol, model=model,
                     trace_mode=si.FULL), o


def test_invariants_random_micro_configs(oracle_lib):
    rng = np.random.default_rng(2024)
    for _ in range(150):
        cfg, o = _random_micro(rng)
        r = _sim(cfg, want=("summary", "records", "iters", "trace"))
        s, rec = r["summary"], r["records"]
        fin = rec["status"] == 1
        assert s["n_finished"] + s["n_rejected"] == len(rec)
        assert s["n_request_iterations"] == int(o[fin].sum())
        assert (rec["e2e_ns"][fin] >= rec["ttft_ns"][fin]).all()
        first = rec["ttft_ns"][fin] + np.asarray(cfg.workload.trace_arrival_ns)[fin]
        assert (np.diff(first) >= 0).all()                                   # S:392 FCFS
        tr = r["trace"][0]
        assert (tr["blocks_max"] <= s["total_blocks"]).all()
        assert int(tr["block_ns"].sum()) == s["block_ns_sum"]
        if cfg.policies[0].kind != si.CONT_RATIO:
            assert s["n_rejected"] == 0


def test_binned_trace_integral_equals_full(oracle_lib):
    cfg = replace(si.c1(), options=si.Options(trace_mode=si.BINNED, trace_bin_ns=250_000_000))
    from oracle import oracle as O
    rb = O.simulate(cfg, 0, want=("summary", "trace"))
    rf = O.simulate(replace(cfg, options=si.Options(trace_mode=si.FULL, trace_cap_bytes=1 << 24)), 0,
                    want=("summary", "trace", "iters"))
    assert int(rb["trace"][0]["block_ns"].sum()) == int(rf["trace"][0]["block_ns"].sum()) == rb["summary"]["block_ns_sum"]
    assert len(rb["trace"][0]) == -(-rb["summary"]["t_final"] // 250_000_000)
    assert int(rb["trace"][0]["n_iter"].sum()) == rb["summary"]["n_iterations"]
    assert rb["trace"][0]["blocks_max"].max() == rb["summary"]["peak_blocks"]


def test_nearest_rank_quantiles(oracle_lib):
    """nearest rank = ceil(q*n)-th smallest.  Isolated o=1 requests have
    e2e = T_pre(p) exactly, so the latency multiset is known in closed form."""
    ps = [int(x) for x in np.random.default_rng(3).permutation(np.arange(5, 105))]
    cfg = trace_cfg([(i * 10 ** 11, p, 1) for i, p in enumerate(ps)])
    r = _sim(cfg)
    lat = sorted(_t(cfg, prefills=[p]) / 1e9 for p in ps)
    st = r["summary"]["stat"]
    for j, q in enumerate((0.50, 0.90, 0.99, 1.00)):
        assert st[2][j] == lat[math.ceil(q * len(lat)) - 1]
    assert st[2][3] == max(lat) and st[1].tolist() == [0.0] * 5     # o = 1: TPOT excluded
    assert abs(st[2][4] - sum(lat) / len(lat)) < 1e-12


def test_goodput_definition(oracle_lib):
    cfg = replace(si.c1(), workload=replace(si.c1().workload, rates=[40.0]),
                  options=si.Options(slo_ttft_s=0.06, slo_mtpot_s=0.08))
    from oracle import oracle as O
    r = O.simulate(cfg, 0)
    rec, s = r["records"], r["summary"]
    a, p, o = O.workload(cfg, 0)
    fin = rec["status"] == 1
    span = (int((rec["e2e_ns"] + a)[fin].max()) - int(a[0])) / 1e9
    ok_mt = fin & (rec["mtpot_ns"] <= 80_000_000)
    ok_both = ok_mt & (rec["ttft_ns"] <= 60_000_000)
    assert 0 < ok_both.sum() < ok_mt.sum() < fin.sum()
    assert s["goodput_mtpot_rps"] == pytest.approx(ok_mt.sum() / span, rel=1e-12)
    assert s["goodput_both_rps"] == pytest.approx(ok_both.sum() / span, rel=1e-12)
    assert s["throughput_rps"] == pytest.approx(fin.sum() / span, rel=1e-12)


def test_finding1_continuous_beats_static(oracle_lib):
    """Finding 1 as a trend check: NORM latency P50/P99 of continuous
    batching <= static batching at every rate, and the gap grows with load."""
    from oracle import oracle as O
    gaps = []
    for lam in (1.0, 2.0, 4.0):
        w = si.Workload(2000, [lam], [0])
        out = {}
        for k in (si.STATIC, si.CONT):
            cfg = si.SweepConfig("f1", si.LLAMA2_7B, [si.A100], [si.Policy(kind=k, max_num_seqs=16)], w)
            out[k] = O.simulate(cfg, 0)["summary"]["stat"][3]
        assert out[si.CONT][0] <= out[si.STATIC][0] and out[si.CONT][2] <= out[si.STATIC][2]
        gaps.append(out[si.STATIC][0] - out[si.CONT][0])
    assert gaps[0] < gaps[-1]


def test_finding2_ratio_reduces_preemption(oracle_lib):
    """Finding 2: limiting new-request admission to a memory ratio reduces
    preemptions on a preemption-heavy scenario."""
    from oracle import oracle as O
    w = si.Workload(1500, [12.0], [0])
    res = {}
    for r in (1.0, 0.7):
        k = si.CONT_RATIO if r < 1 else si.CONT
        cfg = si.SweepConfig("f2", si.LLAMA2_13B, [si.A100], [si.Policy(kind=k, max_mem_ratio=r)], w)
        res[r] = O.simulate(cfg, 0)["summary"]
    assert res[1.0]["n_preemptions"] > 0
    assert res[0.7]["n_preemptions"] < res[1.0]["n_preemptions"]
    assert res[0.7]["stat"][4][3] < res[1.0]["stat"][4][3]         # max mTPOT shrinks


# ------------------------------------------------------------------ a.9 P/D pair
def _pd_cfg(reqs, hwP=si.A100_IDEAL, hwD=None, pol=si.Policy(), model=si.LLAMA2_7B, **opt):
    hwD = hwD or replace(si.A100_IDEAL, mem_bw=4e12)
    w = si.Workload(len(reqs), [1.0], [0], len_dist=si.TRACE, trace_arrival_ns=[r[0] for r in reqs],
                    trace_prompt=[r[1] for r in reqs], trace_output=[r[2] for r in reqs],
                    prompt_table=None, output_table=None)
    return si.SweepConfig("pd", model, [hwP, hwD], [pol], w, si.Options(topology=si.PD_PAIR, **opt))


def _pd_sim(cfg, **kw):
    from oracle import oracle as O
    return O.simulate(cfg, 1, check_invariants=True, **kw)  # point 1 = (P = hw0, D = hw1)


def _xfer_ns(p, kvb=524288, bw=200e9):
    return math.floor(p * kvb / bw * 1e9 + 0.5)


def test_pd_isolated_requests_closed_form(oracle_lib):
    """Isolated requests: e2e = T_pre on P + KV transfer p*kvb/link + decode
    steps on D; mTPOT includes the transfer in the first decode gap; P frees its blocks when
    the transfer ends (A35)."""
    from oracle import oracle as O
    reqs = [(0, 20, 3), (10 ** 12, 100, 9), (2 * 10 ** 12, 16, 2), (3 * 10 ** 12, 7, 1)]
    cfg = _pd_cfg(reqs)
    r = _pd_sim(cfg, keep_events=True, want=("summary", "records", "iters", "events"))
    for i, (a, p, o) in enumerate(reqs):
        tp = O.iter_time_ns(cfg, [(p, 0)], [], point=1, decode_worker=0)
        td = [O.iter_time_ns(cfg, [], [p + j], point=1, decode_worker=1) for j in range(1, o)]
        rec = r["records"][i]
        assert rec["ttft_ns"] == tp
        if o == 1:
            assert rec["e2e_ns"] == tp and rec["mtpot_ns"] == 0
        else:
            x = _xfer_ns(p)
            assert rec["e2e_ns"] == tp + x + sum(td)
            assert rec["mtpot_ns"] == max([x + td[0]] + td[1:])
    s = r["summary"]
    assert s["n_transfers"] == 3 and s["transfer_bytes"] == (20 + 100 + 16) * 524288
    assert s["n_request_iterations"] == sum(o for _, _, o in reqs)
    ev = r["events"]
    # request 0: two P blocks allocated by P's first iteration, freed at P's next boundary
    p0 = ev[(ev["req"] == 0) & (ev["worker"] == 0)]
    assert [(int(e["k"]), int(e["kind"]), int(e["block"])) for e in p0] == [(0, 1, 0), (0, 1, 1), (1, 2, 0), (1, 2, 1)]
    d0 = ev[(ev["req"] == 0) & (ev["worker"] == 1)]
    assert [int(e["kind"]) for e in d0] == [1, 1, 2, 2]   # ceil(20/16) blocks pulled, freed at finish


def test_pd_link_is_fifo(oracle_lib):
    """two transfers on one link serialize -- the second completes ~2x later."""
    from oracle import oracle as O
    cfg = _pd_cfg([(0, 64, 2), (0, 64, 2)], pd_link_bw=1e9)   # slow link: transfers dominate
    r = _pd_sim(cfg, want=("summary", "records", "iters"))
    x = _xfer_ns(64, bw=1e9)
    tp = O.iter_time_ns(cfg, [(64, 0), (64, 0)], [], point=1, decode_worker=0)
    rec = r["records"]
    assert rec["ttft_ns"][0] == rec["ttft_ns"][1] == tp
    d1 = O.iter_time_ns(cfg, [], [65], point=1, decode_worker=1)
    assert rec["e2e_ns"][0] == tp + x + d1
    assert rec["e2e_ns"][1] == tp + 2 * x + d1


def _random_pd(rng):
    n = int(rng.integers(1, 50))
    a = np.sort(rng.integers(0, 2_000_000_000, n))
    p = rng.integers(1, 64, n)
    o = rng.integers(1, 64, n)
    mml = 128
    model = replace(si.LLAMA2_7B, max_model_len=mml)
    bs = int(rng.choice([4, 16]))
    mb = -(-mml // bs)
    hwP = replace(si.A100, kv_blocks_override=int(rng.integers(mb, mb + 30)), peak_flops=float(rng.choice([78e12, 312e12])))
    hwD = replace(si.A100, kv_blocks_override=int(rng.integers(mb, mb + 30)), mem_bw=float(rng.choice([1e12, 4e12])))
    pol = si.Policy(kind=str(rng.choice([si.STATIC, si.CONT])), preempt=str(rng.choice([si.SWAP, si.RECOMPUTE])),
                    max_num_seqs=int(rng.choice([2, 8, 256])), block_size=bs)
    return _pd_cfg(list(zip(a.tolist(), p.tolist(), o.tolist())), hwP=hwP, hwD=hwD, pol=pol, model=model,
                   pd_link_bw=float(rng.choice([1e9, 200e9])), trace_mode=si.FULL), p, o


def test_pd_invariants_random(oracle_lib):
    """every finished request with o >= 2 makes exactly one P->D transfer of p*kvb bytes,
    completed before its first decode; conservation on both workers every boundary."""
    rng = np.random.default_rng(99)
    for _ in range(80):
        cfg, p, o = _random_pd(rng)
        r = _pd_sim(cfg, want=("summary", "records", "iters", "trace"))
        s, rec = r["summary"], r["records"]
        assert s["n_finished"] == len(rec) and s["n_request_iterations"] == int(o.sum())
        multi = o >= 2
        assert s["n_transfers"] == int(multi.sum()) and s["transfer_bytes"] == int(p[multi].sum()) * 524288
        for i in np.nonzero(multi)[0]:
            assert rec["mtpot_ns"][i] >= _xfer_ns(int(p[i]), bw=cfg.options.pd_link_bw)
        it = r["iters"]
        assert (it["S_p"][it["worker"] == 0] == it["n_admitted"][it["worker"] == 0]).all()   # P: prefill only
        if cfg.policies[0].preempt == si.SWAP:
            assert (it["S_p"][it["worker"] == 1] == 0).all()   # D: no prefill except RECOMPUTE (A35)


def test_pd_finding5_prefill_footprint(oracle_lib):
    """Finding 5: prefill-side KV footprint is much lower than decode-side."""
    from oracle import oracle as O
    w = si.Workload(1500, [6.0], [0], len_dist=si.FIXED, prompt_a=128, output_a=1024)
    cfg = si.SweepConfig("pdfp", si.LLAMA2_7B, [si.A100, si.A100], [si.Policy()], w,
                         si.Options(topology=si.PD_PAIR, trace_bin_ns=1_000_000_000))
    r = O.simulate(cfg, 1, want=("summary", "trace"))
    tp, td = r["trace"]
    sel = slice(5, 65)   # the paper's [5, 65] s window
    uP = tp["block_ns"][sel].sum() / O.derive(cfg, 1, 0)["total_blocks"]
    uD = td["block_ns"][sel].sum() / O.derive(cfg, 1, 1)["total_blocks"]
    assert uP < 0.5 * uD


# ------------------------------------------------------------------ NEXT-3 prefill-first iterations
def test_prefill_first_two_request_trace(oracle_lib):
    """vLLM v0.6.2 default (ext, reading R-N3): an admissible fresh request gets a prefill-only
    iteration and the running request pauses, so its next token gap spans that iteration."""
    reqs = [(0, 20, 3), (1_000_000, 10, 2)]
    cfg = trace_cfg(reqs, pol=si.Policy(iteration_mode=si.PREFILL_FIRST))
    r = _sim(cfg, want=("summary", "records", "iters"))
    it, rec = r["iters"], r["records"]
    t_pre20, t_pre10 = _t(cfg, prefills=[20]), _t(cfg, prefills=[10])
    t_d = _t(cfg, decodes=[21, 11])
    t_d2 = _t(cfg, decodes=[22])
    assert list(it["T_ns"]) == [t_pre20, t_pre10, t_d, t_d2]
    assert list(it["S_p"]) == [1, 1, 0, 0] and list(it["D"]) == [0, 0, 2, 1]
    assert rec["ttft_ns"][0] == t_pre20
    assert rec["ttft_ns"][1] == t_pre20 + t_pre10 - 1_000_000
    assert rec["e2e_ns"][1] == t_pre20 + t_pre10 + t_d - 1_000_000
    assert rec["e2e_ns"][0] == t_pre20 + t_pre10 + t_d + t_d2
    assert rec["mtpot_ns"][0] == max(t_pre10 + t_d, t_d2)       # the paused iteration counts
    mixed = _sim(trace_cfg(reqs), want=("summary", "iters"))
    assert mixed["summary"]["n_iterations"] == 3


def test_prefill_first_iteration_shapes(oracle_lib):
    """Every prefill-first iteration is either prefill-only (fresh admissions, no decodes) or a
    decode iteration with no fresh admission; invariants hold on random micro configs."""
    rng = np.random.default_rng(31)
    for _ in range(60):
        cfg, o = _random_micro(rng)
        cfg = replace(cfg, policies=[replace(cfg.policies[0], iteration_mode=si.PREFILL_FIRST)])
        r = _sim(cfg, want=("summary", "records", "iters"))
        it, s = r["iters"], r["summary"]
        pf = it["n_admitted"] > 0
        assert (it["D"][pf] == 0).all() and (it["S_p"][pf] == it["n_admitted"][pf]).all()
        assert (it["n_admitted"][~pf] == 0).all()
        fin = r["records"]["status"] == 1
        assert s["n_request_iterations"] == int(o[fin].sum()) and s["n_finished"] + s["n_rejected"] == len(o)


# ------------------------------------------------------------------ NEXT-3b chunked prefill
def _tc(cfg, prefills=(), decodes=()):
    """Cost of a batch with explicit chunks (P, c0, emits)."""
    from oracle import oracle as O
    return O.iter_time_ns(cfg, list(prefills), decodes, 0)


@pytest.mark.parametrize("model", [si.LLAMA2_7B, si.LLAMA2_70B])
def test_chunk_cost_limits(oracle_lib, model):
    """A chunk of L tokens after c0 computed ones (c.5 with c0 > 0): compute-bound it costs
    2 FLOPs per linear weight per token plus causal attention 4*q*Lyr*(L*c0 + L(L+1)/2), plus the
    LM-head row only if it emits; memory-bound each prefix token adds exactly kvb bytes."""
    pub = gold("llama2_published.json")["models"][model.name]
    F, B = 312e12, 2.039e12
    cfg_f = _one(model, si.Hw(peak_flops=F, mem_bw=1e30, eff_flops=1, eff_bw=1, iter_overhead_s=0,
                              mem_capacity=10 ** 12))
    cfg_b = _one(model, si.Hw(peak_flops=1e30, mem_bw=B, eff_flops=1, eff_bw=1, iter_overhead_s=0,
                              mem_capacity=10 ** 12))
    L, h, V = model.num_layers, model.hidden, model.vocab
    q = model.num_heads * model.head_dim
    linear = pub["params"] - 2 * V * h - (2 * L + 1) * h
    for P, c0 in ((1, 0), (16, 16), (512, 1536), (100, 7)):
        for emits in (True, False):
            flops = 2 * P * linear + 4 * q * L * (P * c0 + P * (P + 1) // 2) + (2 * h * V if emits else 0)
            assert abs(_tc(cfg_f, [(P, c0, emits)]) - flops / F * 1e9) <= 2
    # the causal-attention FLOPs of the chunks of one prompt add up to the whole prompt's
    chunks = [(16, 0, False), (16, 16, False), (8, 32, True)]
    att = sum(4 * q * L * (P * c0 + P * (P + 1) // 2) for P, c0, _ in chunks)
    assert att == 4 * q * L * 40 * 41 // 2
    d = _tc(cfg_b, [(1, 1001, False)]) - _tc(cfg_b, [(1, 1, False)])
    assert abs(d - 1000 * pub["kvb"] / B * 1e9) <= 2


def test_chunked_single_request_trace(oracle_lib):
    """Budget 16 (R-N3b): a 40-token prompt runs as chunks 16 + 16 + 8; only the last emits the
    first token; then two decodes."""
    pol = si.Policy(iteration_mode=si.CHUNKED, max_batched_tokens=16, max_num_seqs=8)
    cfg = trace_cfg([(0, 40, 3)], pol=pol)
    r = _sim(cfg, want=("summary", "records", "iters"))
    it, rec, s = r["iters"], r["records"][0], r["summary"]
    T = [_tc(cfg, [(16, 0, False)]), _tc(cfg, [(16, 16, False)]), _tc(cfg, [(8, 32, True)]),
         _tc(cfg, decodes=[41]), _tc(cfg, decodes=[42])]
    assert list(it["T_ns"]) == T
    assert list(it["S_p"]) == [1, 1, 1, 0, 0] and list(it["D"]) == [0, 0, 0, 1, 1]
    assert list(it["N_p"]) == [16, 16, 8, 0, 0]
    assert rec["ttft_ns"] == sum(T[:3]) and rec["e2e_ns"] == sum(T) and rec["mtpot_ns"] == max(T[3:])
    assert s["n_request_iterations"] == 5


def test_chunked_two_request_budget_split(oracle_lib):
    """Decodes take the budget first, then the prefill in progress, then new arrivals (vLLM v0.6.2
    chunked-prefill order): r0 decodes while r1's 30-token prompt is chunked 15 + 15 under a
    budget of 16."""
    pol = si.Policy(iteration_mode=si.CHUNKED, max_batched_tokens=16, max_num_seqs=4)
    cfg = trace_cfg([(0, 8, 4), (0, 30, 2)], pol=pol)
    r = _sim(cfg, want=("summary", "records", "iters"))
    it, rec = r["iters"], r["records"]
    # k0: r0 prefill 8 (emits) + r1 chunk 8 (budget 16); k1: r0 decode + r1 chunk 15;
    # k2: r0 decode + r1 chunk 7 (emits); k3: r0 decode (finishes) + r1 decode (finishes)
    T = [_tc(cfg, [(8, 0, True), (8, 0, False)]),
         _tc(cfg, [(15, 8, False)], [9]),
         _tc(cfg, [(7, 23, True)], [10]),
         _tc(cfg, decodes=[11, 31])]
    assert list(it["T_ns"]) == T
    assert list(it["N_p"]) == [16, 15, 7, 0] and list(it["D"]) == [0, 1, 1, 2]
    assert list(it["n_admitted"]) == [2, 0, 0, 0]
    assert rec["ttft_ns"][0] == T[0] and rec["ttft_ns"][1] == sum(T[:3])
    assert rec["e2e_ns"][0] == sum(T) and rec["e2e_ns"][1] == sum(T)
    assert rec["mtpot_ns"][0] == max(T[1:]) and rec["mtpot_ns"][1] == T[3]


def test_chunked_unbounded_budget_equals_mixed(oracle_lib):
    """With an unbounded token budget every chunk is the whole prefill, so CHUNKED reduces to
    MIXED (A3) exactly: same iterations, records and summary."""
    rng = np.random.default_rng(77)
    for _ in range(60):
        cfg, _o = _random_micro(rng)
        pol = replace(cfg.policies[0], max_batched_tokens=si.UINT32_MAX)
        a = _sim(replace(cfg, policies=[pol]), want=("summary", "records", "iters"))
        b = _sim(replace(cfg, policies=[replace(pol, iteration_mode=si.CHUNKED)]),
                 want=("summary", "records", "iters"))
        assert repr(a["summary"]) == repr(b["summary"])
        assert a["records"].tobytes() == b["records"].tobytes()
        assert a["iters"].tobytes() == b["iters"].tobytes()


def test_chunked_budget_and_invariants(oracle_lib):
    """Random micro configs under small budgets: every iteration fits the budget (N_p + D <= B),
    held = blocks of the whole target, at most one prefill in progress (checked inside the
    oracle), FCFS first tokens, every request finished or rejected, and prompts longer than the
    budget are served."""
    rng = np.random.default_rng(4242)
    long_served = npre = 0
    for _ in range(120):
        cfg, o = _random_micro(rng)
        pol = cfg.policies[0]
        budget = int(rng.choice([pol.max_num_seqs, 16, 40, 100])) if pol.max_num_seqs <= 16 else \
            int(rng.choice([256, 300]))
        budget = max(budget, min(pol.max_num_seqs, 256))
        pol = replace(pol, iteration_mode=si.CHUNKED, max_batched_tokens=budget)
        cfg = replace(cfg, policies=[pol])
        r = _sim(cfg, want=("summary", "records", "iters"))
        s, rec, it = r["summary"], r["records"], r["iters"]
        assert (it["N_p"].astype(np.int64) + it["D"] <= budget).all()
        fin = rec["status"] == 1
        assert s["n_finished"] + s["n_rejected"] == len(rec)
        assert s["n_request_iterations"] >= int(o[fin].sum())
        assert s["n_request_iterations"] == int((it["S_p"] + it["D"]).sum())
        first = rec["ttft_ns"][fin] + np.asarray(cfg.workload.trace_arrival_ns)[fin]
        assert (np.diff(first) >= 0).all()
        p = np.asarray(cfg.workload.trace_prompt)
        long_served += int((fin & (p > budget)).sum())
        npre += s["n_preemptions"]
        if pol.kind != si.CONT_RATIO:
            assert s["n_rejected"] == 0
    assert long_served > 0 and npre > 0


# ------------------------------------------------------------------ NEXT-1 xP:yD node
def _node(cfg, x, y, dispatch=si.ROUND_ROBIN):
    return replace(cfg, options=replace(cfg.options, pd_prefill=x, pd_decode=y, dispatch=dispatch))


def test_node_1p1d_equals_pair(oracle_lib):
    """With x = y = 1 the general x:y loop (dispatch events, per-worker links) reduces to the
    a.9 pair loop exactly, under every dispatch policy."""
    from oracle import oracle as O
    rng = np.random.default_rng(515)
    for it in range(60):
        cfg, _p, _o = _random_pd(rng)
        if it % 3 == 0:
            cfg = replace(cfg, options=replace(cfg.options, horizon_ns=int(rng.integers(1, 2_000_000_000))))
        a = O.simulate(cfg, 1, check_invariants=True, want=("summary", "records", "iters", "trace"))
        for d in (si.ROUND_ROBIN, si.LEAST_OUTSTANDING, si.LEAST_MEMORY):
            b = O.simulate(_node(cfg, 1, 1, d), 1, check_invariants=True, force_general=True,
                           want=("summary", "records", "iters", "trace"))
            assert repr(a["summary"]) == repr(b["summary"])
            assert a["records"].tobytes() == b["records"].tobytes()
            assert a["iters"].tobytes() == b["iters"].tobytes()
            for w in (0, 1):
                assert a["trace"][w].tobytes() == b["trace"][w].tobytes()


def test_node_round_robin_splits_evenly(oracle_lib):
    """round robin over 3 prefill workers, 6 simultaneous requests -> each gets 2; their
    prefill iterations run concurrently, so every TTFT equals one 2-request prefill."""
    from oracle import oracle as O
    cfg = _node(_pd_cfg([(0, 32, 2)] * 6), 3, 2)
    r = O.simulate(cfg, 1, check_invariants=True, want=("summary", "records", "iters"))
    it = r["iters"]
    first = [it[it["worker"] == w][0] for w in range(3)]
    assert [int(x["S_p"]) for x in first] == [2, 2, 2] and all(int(x["t_start"]) == 0 for x in first)
    tp = O.iter_time_ns(cfg, [(32, 0), (32, 0)], [], point=1, decode_worker=0)
    assert (r["records"]["ttft_ns"] == tp).all()
    # the six completions (same instant, id order) alternate D_0, D_1: three one-decode requests each
    dec = it[it["worker"] >= 3]
    assert sorted(set(dec["worker"].tolist())) == [3, 4]
    assert int(dec[dec["worker"] == 3]["D"].sum()) == 3 and int(dec[dec["worker"] == 4]["D"].sum()) == 3


def test_node_least_outstanding_vs_round_robin(oracle_lib):
    """least-outstanding picks the argmin (ties -> lowest id).  P_0 gets a long prompt,
    P_1 and P_2 short ones; a fourth request arriving after P_1/P_2 finished goes to P_1 under
    least-outstanding (P_0 still busy) but to P_0 under round robin, where it waits."""
    from oracle import oracle as O
    reqs = [(0, 2000, 2), (0, 8, 2), (0, 8, 2), (60_000_000, 8, 2)]
    base = _pd_cfg(reqs, model=replace(si.LLAMA2_7B, max_model_len=4096))
    t_long = O.iter_time_ns(base, [(2000, 0)], [], point=1, decode_worker=0)
    t_short = O.iter_time_ns(base, [(8, 0)], [], point=1, decode_worker=0)
    assert t_short < 60_000_000 < t_long
    lo = O.simulate(_node(base, 3, 1, si.LEAST_OUTSTANDING), 1, check_invariants=True, want=("records", "iters"))
    rr = O.simulate(_node(base, 3, 1, si.ROUND_ROBIN), 1, check_invariants=True, want=("records", "iters"))
    assert lo["records"]["ttft_ns"][3] == t_short
    assert rr["records"]["ttft_ns"][3] == t_long - 60_000_000 + t_short
    assert 1 in lo["iters"][lo["iters"]["t_start"] == 60_000_000]["worker"].tolist()


def test_node_least_memory_prefers_empty_worker(oracle_lib):
    """S:387 least-memory: a decode worker holding a long context is avoided; the argmin of
    allocated blocks (ties -> lowest id) receives the next request."""
    from oracle import oracle as O
    reqs = [(0, 1000, 400), (500_000_000, 16, 4)]
    base = _pd_cfg(reqs, model=replace(si.LLAMA2_7B, max_model_len=2048))
    lm = O.simulate(_node(base, 1, 2, si.LEAST_MEMORY), 1, check_invariants=True, want=("iters",))
    rr = O.simulate(_node(base, 1, 2, si.ROUND_ROBIN), 1, check_invariants=True, want=("iters",))
    # both send r1 to D_1 (RR: second completion; LM: D_0 holds r0's blocks) ...
    for r in (lm, rr):
        it = r["iters"]
        assert int(it[it["worker"] == 2]["D"].max()) == 1
    # ... while with 3 requests RR returns to D_0 and LM keeps avoiding it
    reqs3 = reqs + [(900_000_000, 16, 4)]
    b3 = _pd_cfg(reqs3, model=replace(si.LLAMA2_7B, max_model_len=2048))
    lm3 = O.simulate(_node(b3, 1, 2, si.LEAST_MEMORY), 1, check_invariants=True, want=("iters",))
    rr3 = O.simulate(_node(b3, 1, 2, si.ROUND_ROBIN), 1, check_invariants=True, want=("iters",))
    assert int(rr3["iters"][rr3["iters"]["worker"] == 1]["D"].max()) == 2
    assert int(lm3["iters"][lm3["iters"]["worker"] == 1]["D"].max()) == 1


def test_node_isolated_requests_match_pair(oracle_lib):
    """Requests far apart never interact, so every x:y node gives the 1:1 pair's latencies
    (finish_k differs: iteration indices are per worker)."""
    from oracle import oracle as O
    reqs = [(k * 10 ** 12, 20 + 7 * k, 1 + k % 5) for k in range(8)]
    pair = O.simulate(_pd_cfg(reqs), 1, want=("records",))["records"]
    fields = ["ttft_ns", "e2e_ns", "mtpot_ns", "n_preempt", "status"]
    for x, y in ((2, 2), (3, 5), (7, 1), (1, 7)):
        for d in (si.ROUND_ROBIN, si.LEAST_OUTSTANDING, si.LEAST_MEMORY):
            got = O.simulate(_node(_pd_cfg(reqs), x, y, d), 1, check_invariants=True, want=("records",))["records"]
            for f in fields:
                assert (got[f] == pair[f]).all(), f


def test_node_invariants_random(oracle_lib):
    """Random x:y nodes: conservation per worker and every decode on one worker (checked
    inside the oracle), one transfer per finished request with o >= 2, request-iterations = sum o,
    prefill workers run prefill-only iterations, and per-worker iteration indices are dense."""
    from oracle import oracle as O
    rng = np.random.default_rng(616)
    for _ in range(60):
        cfg, p, o = _random_pd(rng)
        x = int(rng.integers(1, 5))
        y = int(rng.integers(1, 9 - x))
        d = str(rng.choice([si.ROUND_ROBIN, si.LEAST_OUTSTANDING, si.LEAST_MEMORY]))
        cfg = _node(cfg, x, y, d)
        r = O.simulate(cfg, 1, check_invariants=True, want=("summary", "records", "iters", "trace"))
        s, rec, it = r["summary"], r["records"], r["iters"]
        assert s["n_finished"] == len(rec) and s["n_request_iterations"] == int(o.sum())
        multi = o >= 2
        assert s["n_transfers"] == int(multi.sum())
        pw = it["worker"] < x
        assert (it["S_p"][pw] == it["n_admitted"][pw]).all() and (it["D"][pw] == 0).all()
        for w in range(x + y):
            k = it["k"][it["worker"] == w]
            assert (k == np.arange(len(k))).all()
        assert len(r["trace"]) == x + y
        assert s["total_blocks"] == y * O.derive(cfg, 1, 1)["total_blocks"]


# ------------------------------------------------------------------ NEXT-4 preload-buffer link
def _brute_pipeline(n, a, b, K):
    """Tick-by-tick simulation of a producer/consumer pair with a K-chunk buffer (integer
    durations): a chunk occupies a slot from its load start until the consumer takes it; at each
    tick finished work completes first, then the consumer takes the next loaded chunk, then the
    producer starts the next load if a slot is free."""
    t = 0
    loaded = 0            # chunks fully loaded
    taken = 0             # chunks the consumer has started
    load_end = None       # end tick of the load in progress
    cons_end = None       # end tick of the chunk being consumed
    done = 0
    while done < n:
        if load_end is not None and load_end == t:
            loaded += 1
            load_end = None
        if cons_end is not None and cons_end == t:
            done += 1
            cons_end = None
        if cons_end is None and taken < loaded:
            taken += 1
            cons_end = t + b
        in_buf = loaded - taken + (1 if load_end is not None else 0)
        started = loaded + (1 if load_end is not None else 0)
        if load_end is None and started < n and in_buf < K:
            load_end = t + a
        if done == n:
            return t
        t += 1
    return t


def test_preload_pipeline_brute_force(oracle_lib):
    """S:444 property test: the oracle's pipeline recurrence equals a step-by-step simulation."""
    from oracle import oracle as O
    rng = np.random.default_rng(8)
    for _ in range(400):
        n, a, b, K = (int(rng.integers(1, 12)), int(rng.integers(1, 9)), int(rng.integers(1, 9)),
                      int(rng.integers(1, 14)))
        assert O.pipeline(n, float(a), float(b), K) == _brute_pipeline(n, a, b, K), (n, a, b, K)


def test_preload_pipeline_closed_forms(oracle_lib):
    """Buffer >= all chunks: the producer never stalls and the two-machine flow shop gives
    max_i(i*a + (n-i+1)*b); one slot with a slower consumer: a + n*b (consumer-governed);
    with a slower link: n*a + b."""
    from oracle import oracle as O
    for n, a, b in ((32, 3.0, 5.0), (32, 5.0, 3.0), (80, 1.0, 1.0), (7, 2.0, 9.0)):
        assert O.pipeline(n, a, b, n) == max(i * a + (n - i + 1) * b for i in range(1, n + 1))
        one = O.pipeline(n, a, b, 1)
        assert one == (a + n * b if a <= b else n * a + b)
        assert one <= n * (a + b)


def test_preload_iteration_never_slower(oracle_lib):
    """with swap-in the PRELOAD iteration is never slower than SEQUENTIAL and is
    non-increasing in the buffer size (strictly faster with a large buffer); without swap-in the
    two modes agree (the swap-out stays serial)."""
    from oracle import oracle as O
    m = si.LLAMA2_13B
    hw = si.Hw(mem_capacity=40 * 10 ** 9, host_link_bw=16e9)
    seq = _one(m, hw)
    L = m.num_layers
    kvb = 2 * L * m.num_kv_heads * m.head_dim * 2
    for blocks in (1, 7, 64):
        swap_in = blocks * 16 * kvb
        t_seq = O.iter_time_ns(seq, [], [300] * 20, 0, swap_in=swap_in)
        prev = t_seq
        for buf in (1, swap_in // L, 4 * swap_in // L, swap_in, 1 << 40):
            c = replace(seq, options=replace(seq.options, link_mode=si.PRELOAD, preload_buffer_bytes=buf))
            t = O.iter_time_ns(c, [], [300] * 20, 0, swap_in=swap_in)
            assert t <= prev + 1
            prev = t
        big = replace(seq, options=replace(seq.options, link_mode=si.PRELOAD, preload_buffer_bytes=1 << 40))
        t_big = O.iter_time_ns(big, [], [300] * 20, 0, swap_in=swap_in)
        assert t_big < t_seq
        c0 = replace(seq, options=replace(seq.options, link_mode=si.PRELOAD, preload_buffer_bytes=1))
        assert O.iter_time_ns(c0, [(64, 0)], [300] * 20, 4096) == O.iter_time_ns(seq, [(64, 0)], [300] * 20, 4096)


def test_preload_simulation_invariants(oracle_lib):
    """Random SWAP-heavy micro configs under a PRELOAD link: the c.8 invariants hold, and a
    config that never swaps in runs exactly as under SEQUENTIAL."""
    rng = np.random.default_rng(909)
    differs = 0
    for _ in range(60):
        cfg, o = _random_micro(rng)
        cfg = replace(cfg, policies=[replace(cfg.policies[0], preempt=si.SWAP)])
        pre = replace(cfg, options=replace(cfg.options, link_mode=si.PRELOAD,
                                           preload_buffer_bytes=int(rng.choice([1, 1 << 16, 1 << 30]))))
        a = _sim(cfg, want=("summary", "records"))
        b = _sim(pre, want=("summary", "records"))
        s = b["summary"]
        assert s["n_finished"] + s["n_rejected"] == len(o)
        if a["summary"]["swap_in_bytes"] == 0:
            assert a["records"].tobytes() == b["records"].tobytes()
        else:
            differs += a["records"].tobytes() != b["records"].tobytes()
    assert differs > 0


# ------------------------------------------------------------------ NEXT-2 multi-round + memory cache
def _mr_cfg(n=1, seed=0, rate=1.0, len_dist=si.FIXED, pa=64, oa=16, cache=True, mml=4096, cap=0,
            think=5.0, pol=si.Policy(), hw=si.A100, **wkw):
    w = si.Workload(n, [rate], [seed], len_dist=len_dist, prompt_a=pa, prompt_b=wkw.pop("pb", 0),
                    output_a=oa, output_b=wkw.pop("ob", 0), multi_round=True, think_mean_s=think, **wkw)
    return si.SweepConfig("mr", replace(si.LLAMA2_7B, max_model_len=mml), [hw], [pol], w,
                          si.Options(memory_cache=cache, cache_capacity_blocks=cap))


def test_rounds_workload_statistics(oracle_lib):
    """half the conversations are single-round, the rest uniform over 2..7 rounds;
    think gaps are Exp(mean 5 s); round r's prompt is the prior context plus a new turn drawn
    from the prompt distribution; round 0 is exactly the a.1 stream."""
    from oracle import oracle as O
    from scipy import stats
    cfg = _mr_cfg(n=20000, seed=3, len_dist=si.UNIFORM, pa=10, pb=50, oa=5, ob=20, mml=1 << 16)
    at, P, Oo, cv = O.workload_rounds(cfg)
    rounds = np.bincount(cv, minlength=20000)
    single = (rounds == 1).mean()
    assert abs(single - 0.5) < 5 * math.sqrt(0.25 / 20000)
    multi = rounds[rounds > 1]
    cnt = np.bincount(multi, minlength=8)[2:8]
    assert stats.chisquare(cnt).pvalue > 1e-4
    first = np.r_[True, cv[1:] != cv[:-1]]
    a0, p0, o0 = O.workload(cfg)
    assert (at[first] == a0).all() and (P[first] == p0).all() and (Oo[first] == o0).all()
    gaps = at[~first] / 1e9
    assert abs(gaps.mean() - 5.0) / 5.0 < 0.03
    assert stats.kstest(gaps, "expon", args=(0, 5.0)).pvalue > 1e-4
    idx = np.nonzero(~first)[0]
    q = P[idx].astype(np.int64) - P[idx - 1] - Oo[idx - 1]
    assert q.min() >= 10 and q.max() <= 50 and abs(q.mean() - 30) < 0.5
    assert ((Oo >= 5) & (Oo <= 20)).all()


def test_rounds_context_cap(oracle_lib):
    """A round whose prompt (prior context + new turn) leaves no room for one output token ends
    its conversation; every kept round satisfies P + o <= max_model_len."""
    from oracle import oracle as O
    cfg = _mr_cfg(n=3000, seed=1, len_dist=si.UNIFORM, pa=100, pb=400, oa=50, ob=300, mml=1024)
    at, P, Oo, cv = O.workload_rounds(cfg)
    assert (P.astype(np.int64) + Oo <= 1024).all() and (Oo >= 1).all()
    rounds = np.bincount(cv)
    assert rounds.max() < 7    # contexts outgrow 1024 tokens before 7 rounds


def _two_round_seed():
    from oracle import oracle as O
    for seed in range(200):
        at, P, Oo, cv = O.workload_rounds(_mr_cfg(seed=seed))
        if len(P) >= 2:
            return seed, at, P, Oo
    raise AssertionError("no multi-round seed")


def test_memory_cache_hand_trace(oracle_lib):
    """One conversation, isolated rounds: round r >= 1 arrives its think gap after round r-1
    finishes; with the cache its prefill is the (P - c0, c0) row, c0 = P_{r-1} + o_{r-1} - 1, plus
    800 ns per cached block; without the cache it re-prefills all P tokens."""
    from oracle import oracle as O
    seed, at, P, Oo = _two_round_seed()
    on = _mr_cfg(seed=seed)
    off = _mr_cfg(seed=seed, cache=False)
    ron = O.simulate(on, 0, check_invariants=True, want=("summary", "records", "iters"))
    roff = O.simulate(off, 0, check_invariants=True, want=("summary", "records", "iters"))
    # round 0 is identical
    assert ron["records"][0].tobytes() == roff["records"][0].tobytes()
    c0 = int(P[0] + Oo[0] - 1)
    t_hit = O.iter_time_ns(on, [(int(P[1]) - c0, c0)], [])
    t_miss = O.iter_time_ns(off, [(int(P[1]), 0)], [])
    blocks = -(-c0 // 16)
    assert abs(ron["records"]["ttft_ns"][1] - (t_hit + 800 * blocks)) <= 1
    assert roff["records"]["ttft_ns"][1] == t_miss
    fin0 = ron["records"]["e2e_ns"][0] + at[0]
    it1 = ron["iters"][ron["iters"]["t_start"] >= fin0]
    assert int(it1["t_start"][0]) == fin0 + at[1]   # causality: arrival = finish + think
    assert int(it1["N_p"][0]) == int(P[1]) - c0


def test_memory_cache_prefill_work(oracle_lib):
    """the cache can only reduce prefill work.  With SWAP preemption every admitted round
    r >= 1 hits a large cache, so total prefill tokens = sum of round-0 prompts + sum over later
    rounds of (new turn + 1); a cache too small for any context changes nothing at all."""
    from oracle import oracle as O
    for seed in range(3):
        base = _mr_cfg(n=60, seed=seed, rate=4.0, len_dist=si.UNIFORM, pa=16, pb=128, oa=4, ob=64,
                       think=0.5, pol=si.Policy(preempt=si.SWAP))
        at, P, Oo, cv = O.workload_rounds(base)
        first = np.r_[True, cv[1:] != cv[:-1]]
        idx = np.nonzero(~first)[0]
        expect = int(P[first].sum()) + int((P[idx].astype(np.int64) - P[idx - 1] - Oo[idx - 1] + 1).sum())
        big = replace(base, options=replace(base.options, cache_capacity_blocks=1 << 40))
        rb = O.simulate(big, 0, check_invariants=True, want=("summary", "iters"))
        assert rb["summary"]["n_finished"] == len(P)
        assert int(rb["iters"]["N_p"].sum()) == expect
        off = O.simulate(replace(base, options=replace(base.options, memory_cache=False)), 0,
                         want=("summary", "records", "iters"))
        assert int(off["iters"]["N_p"].sum()) == int(P.sum()) >= expect
        tiny = O.simulate(replace(base, options=replace(base.options, cache_capacity_blocks=1)), 0,
                          want=("summary", "records"))
        assert tiny["records"].tobytes() == off["records"].tobytes()


def test_memory_cache_invariants_random(oracle_lib):
    """Random multi-round configs (all policies, both preemption modes, LRU capacities):
    conservation and cache accounting every iteration, every request finished or rejected."""
    from oracle import oracle as O
    rng = np.random.default_rng(321)
    for _ in range(40):
        bs = int(rng.choice([4, 16]))
        total = int(rng.integers(-(-512 // bs), -(-512 // bs) + 60))
        pol = si.Policy(kind=str(rng.choice([si.STATIC, si.CONT, si.CONT_RATIO])),
                        preempt=str(rng.choice([si.SWAP, si.RECOMPUTE])), max_mem_ratio=0.8,
                        max_num_seqs=int(rng.choice([2, 8, 256])), block_size=bs)
        cfg = _mr_cfg(n=int(rng.integers(1, 40)), seed=int(rng.integers(0, 1000)), rate=float(rng.choice([1.0, 8.0])),
                      len_dist=si.UNIFORM, pa=8, pb=120, oa=2, ob=60, mml=512, think=float(rng.choice([0.05, 1.0])),
                      cap=int(rng.choice([0, 8, 64])), pol=pol, hw=replace(si.A100, kv_blocks_override=total))
        r = O.simulate(cfg, 0, check_invariants=True, want=("summary", "records"))
        s = r["summary"]
        assert s["n_finished"] + s["n_rejected"] == s["n_requests"] == len(r["records"])


def test_finding6_cache_helps_short_outputs(oracle_lib):
    """Finding 6: at a high request rate the memory cache lowers P99 latency of
    multi-round conversations with ~64-token outputs."""
    from oracle import oracle as O
    res = {}
    for cache in (False, True):
        cfg = _mr_cfg(n=400, seed=7, rate=12.0, len_dist=si.UNIFORM, pa=200, pb=600, oa=32, ob=96,
                      think=1.0, cache=cache, mml=4096)
        s = O.simulate(cfg, 0, want=("summary",))["summary"]
        res[cache] = s["stat"][2][2]   # E2E P99
    assert res[True] < res[False]
