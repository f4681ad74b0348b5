"""CUDA path vs oracle, element by element, through the C ABI (-m gpu).

Bar (BASELINE.json north_star): schedules, batch compositions, preemptions, block ids and
per-request token counts bit-exact (digests + records + iteration traces); fp64
latencies/quantiles within 1e-9 relative (expected equal: both sides evaluate the same
fp64 expressions in the same order without FMA)."""
import os
from dataclasses import replace

import numpy as np
import pytest

import sweep_inputs as si

from parity import (compare_iters, compare_records, compare_summary, compare_trace, oracle_points,
                    sample_points)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_08415_b200 import build
    build.build()
    import paper_2503_08415_b200 as P
    return P


def run_gpu(api, cfg, begin=0, end=None, stride=1):
    sw = api.Sweep(cfg)
    sw.run(begin, end, stride)
    return sw


def check_points(sw, cfg, points, records=True, trace=False, iters=False):
    want = ["summary"] + (["records"] if records else []) + (["trace"] if trace else []) + \
           (["iters"] if iters else [])
    ora = oracle_points(cfg, points, want=tuple(want))
    bad = []
    full = cfg.options.trace_mode == si.FULL
    for p in points:
        o = ora[p]
        g = sw.summary(p)
        bad += compare_summary(g, o["summary"], p, full_trace=full)
        if records:
            bad += compare_records(sw.records(p), o["records"], p)
        if trace:
            bad += compare_trace(sw.mem_trace(p), o["trace"][0], p, prefix=full and bool(int(g["status_flags"]) & 1))
        if iters:
            bad += compare_iters(sw.iteration_trace(p), o["iters"], p)
    assert not bad, "\n".join(bad[:20])


def test_c1_bit_exact(api):
    cfg = replace(si.c1(), options=si.Options(iteration_trace_cap=1 << 20))
    sw = run_gpu(api, cfg)
    check_points(sw, cfg, [0], records=True, trace=True, iters=True)


def test_workload_generator(api):
    from oracle import oracle as O
    cfg = si.c2()
    sw = run_gpu(api, cfg)
    for p in (0, 7, 63, 64, 127):
        ga, gp, go = sw.workload(p)
        oa, op, oo = O.workload(cfg, p)
        assert (ga == oa).all() and (gp == op).all() and (go == oo).all(), p


def test_c2_every_point(api):
    cfg = si.c2()
    sw = run_gpu(api, cfg)
    check_points(sw, cfg, list(range(cfg.num_points)), records=True)


def test_c2_sharding_invariance(api):
    cfg = si.c2()
    full = run_gpu(api, cfg).summaries()
    for b, s in ((1, 3), (2, 5), (0, 8)):
        part = run_gpu(api, cfg, b, None, s).summaries()
        ref = full[b::s]
        assert part.tobytes() == np.ascontiguousarray(ref).tobytes(), (b, s)


def test_lean_kernel_variants_agree(api):
    """More points than SMs run the compact lean kernel (several warps per SM, variant 4); a
    strided run of at most one point per SM runs the inline one (variant 0).  Same bytes, and a
    non-power-of-two block size (the general block arithmetic instantiation) agrees too."""
    for bs in (16, 12):
        cfg = replace(si.c2(n_seeds=24), policies=[si.Policy(block_size=bs)])
        assert cfg.num_points > 148
        full = run_gpu(api, cfg)
        s = full.summaries()
        for b in range(3):
            part = run_gpu(api, cfg, b, None, 3)
            assert part.summaries().tobytes() == np.ascontiguousarray(s[b::3]).tobytes(), (bs, b)
            for p in (b, b + 3 * 40):
                assert part.records(p).tobytes() == full.records(p).tobytes(), (bs, p)
        check_points(full, cfg, [0, 200, cfg.num_points - 1], records=True)


def test_kernel_variants_byte_identical(api, monkeypatch):
    """The same 384-point sweep through the three lean kernels the host chooses between --
    8 independent warps per SM (variant 4), the helper-warp kernel without (variant 5) and with
    (variant 0) extended stretches -- and through other queue orders and launch shapes gives
    identical bytes (summaries, records)."""
    cfg = si.c2(n_seeds=24)
    runs = {}
    for name, env in (("auto", {}), ("v4", {"TOKENSIM_HELPER": "0"}), ("v0", {"TOKENSIM_XS": "1"}),
                      ("v5", {"TOKENSIM_XS": "0"}), ("v4-old-order", {"TOKENSIM_HELPER": "0", "TOKENSIM_LPT_OLD": "1"}),
                      ("v4-wpb2", {"TOKENSIM_HELPER": "0", "TOKENSIM_WPB": "2", "TOKENSIM_BPS": "3"}),
                      ("v4-six", {"TOKENSIM_HELPER": "0", "TOKENSIM_WPB": "3", "TOKENSIM_BPS": "2"})):
        for k in ("TOKENSIM_HELPER", "TOKENSIM_XS", "TOKENSIM_LPT_OLD", "TOKENSIM_WPB", "TOKENSIM_BPS"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        sw = run_gpu(api, cfg)
        runs[name] = (sw, sw.run_info()["helper_mode"])
    for k in ("TOKENSIM_HELPER", "TOKENSIM_XS", "TOKENSIM_LPT_OLD", "TOKENSIM_WPB", "TOKENSIM_BPS"):
        monkeypatch.delenv(k, raising=False)
    assert runs["v4"][1] == 0 and runs["v0"][1] == 1 and runs["v5"][1] == 2 and runs["auto"][1] == 2
    ref = runs["auto"][0]
    for name, (sw, _) in runs.items():
        assert sw.summaries().tobytes() == ref.summaries().tobytes(), name
        for p in (0, 191, 383):
            assert sw.records(p).tobytes() == ref.records(p).tobytes(), (name, p)


def test_full_kernel_helper_variant_byte_identical(api, monkeypatch):
    """The full kernel with (variant 6) and without (variant 1) the helper warp gives identical
    bytes -- summaries, records, iteration records and memory traces -- on multi-round
    conversations with the memory cache (c7-shaped, small), on prefill-first / chunked
    iterations under memory pressure, FULL and BINNED traces, SWAP and RECOMPUTE, and on
    SWAP-heavy points under the preload link (c9-shaped, small)."""
    pols = [si.Policy(preempt=si.SWAP, iteration_mode=si.PREFILL_FIRST),
            si.Policy(preempt=si.RECOMPUTE, iteration_mode=si.CHUNKED, max_batched_tokens=512)]
    cfgs = [
        replace(si.c7(), workload=replace(si.c7().workload, num_requests=300, rates=[0.5, 4.0], seeds=[0, 1]),
                options=replace(si.c7().options, iteration_trace_cap=1 << 16)),
        si.SweepConfig("pf-chunked", si.LLAMA2_13B, [si.Hw(mem_capacity=30 * 10 ** 9), si.A100], pols,
                       si.Workload(300, [4.0, 16.0], [0, 1]),
                       si.Options(trace_mode=si.FULL, iteration_trace_cap=1 << 16)),
        replace(si.c9(), workload=replace(si.c9().workload, num_requests=400, rates=[0.5, 2.0], seeds=[0]),
                options=replace(si.c9().options, iteration_trace_cap=1 << 16)),  # the preload link
    ]
    for cfg in cfgs:
        runs = {}
        for name, v in (("v6", "1"), ("v1", "0")):
            monkeypatch.setenv("TOKENSIM_HELPER", v)
            sw = run_gpu(api, cfg)
            runs[name] = (sw, sw.run_info()["helper_mode"])
        monkeypatch.delenv("TOKENSIM_HELPER", raising=False)
        assert runs["v6"][1] != 0 and runs["v1"][1] == 0
        a, b = runs["v6"][0], runs["v1"][0]
        assert a.summaries().tobytes() == b.summaries().tobytes(), cfg.name
        for p in range(cfg.num_points):
            assert a.records(p).tobytes() == b.records(p).tobytes(), (cfg.name, p)
            assert a.iteration_trace(p).tobytes() == b.iteration_trace(p).tobytes(), (cfg.name, p)
            assert a.mem_trace(p).tobytes() == b.mem_trace(p).tobytes(), (cfg.name, p)


def test_head_reservation_is_byte_identical(api, monkeypatch):
    """TOKENSIM_HEADS=K (the K longest points each get an SM; the other CTAs there leave): every
    queue position is claimed exactly once, so results are byte-identical to the default run."""
    cfg = si.c2(n_seeds=24)
    base = run_gpu(api, cfg)
    for k in (8, 40):
        monkeypatch.setenv("TOKENSIM_HEADS", str(k))
        sw = run_gpu(api, cfg)
        assert sw.run_info()["n_heads"] == k
        assert sw.summaries().tobytes() == base.summaries().tobytes(), k
        for p in (0, 100, 383):
            assert sw.records(p).tobytes() == base.records(p).tobytes(), (k, p)
    monkeypatch.delenv("TOKENSIM_HEADS", raising=False)


def _micro(rng):
    n = int(rng.integers(1, 80))
    a = np.sort(rng.integers(0, 3_000_000_000, n))
    if rng.random() < 0.3:
        a[:] = a[0]  # identical arrival times
    p = rng.integers(1, 64, n)
    if rng.random() < 0.3:
        p = (p // 16 + 1) * 16 % 64 + 16  # p % 16 == 0
    o = rng.integers(1, 64, n)
    if rng.random() < 0.2:
        o[:] = 1
    mml = 128
    model = replace(si.LLAMA2_7B, max_model_len=mml)
    bs = int(rng.choice([1, 4, 16]))
    mb = -(-mml // bs)
    total = int(rng.integers(mb, mb + 40))
    hw = replace(si.A100, kv_blocks_override=total, tp_degree=int(rng.choice([1, 2])), tp_link_bw=300e9)
    pol = si.Policy(kind=str(rng.choice([si.STATIC, si.CONT, si.CONT_RATIO])),
                    preempt=str(rng.choice([si.SWAP, si.RECOMPUTE])),
                    max_mem_ratio=float(rng.choice([0.3, 0.7, 1.0])),
                    max_num_seqs=int(rng.choice([1, 3, 8, 33, 256])), block_size=bs,
                    max_batched_tokens=int(rng.choice([mml, 300, si.UINT32_MAX])),
                    watermark_blocks=int(rng.integers(0, total - mb + 1)))
    w = si.Workload(n, [1.0], [0], len_dist=si.TRACE, trace_arrival_ns=a.tolist(), trace_prompt=p.tolist(),
                    trace_output=o.tolist(), prompt_table=None, output_table=None)
    mode = si.FULL if rng.random() < 0.5 else si.BINNED
    opts = si.Options(trace_mode=mode, trace_bin_ns=int(rng.choice([10_000_000, 1_000_000_000])),
                      iteration_trace_cap=1 << 16, horizon_ns=int(rng.choice([-1, -1, -1, 500_000_000])),
                      fast_forward=bool(rng.random() < 0.8))
    return si.SweepConfig("micro", model, [hw], [pol], w, opts)


def test_adversarial_micro_configs(api):
    """Capacity of a few blocks (preemption storms), max_num_seqs = 1, o = 1, p % 16 == 0,
    identical arrivals, tiny ratios (rejections), STATIC, RECOMPUTE, TP, horizon, FULL trace."""
    rng = np.random.default_rng(7)
    for it in range(60):
        cfg = _micro(rng)
        sw = run_gpu(api, cfg)
        check_points(sw, cfg, [0], records=True, trace=True, iters=True)


def test_preemption_heavy_grid(api):
    """C2-shaped grid squeezed onto a small KV pool: every policy x preemption mode."""
    pols = [si.Policy(kind=k, preempt=pm, max_mem_ratio=r) for k, r in
            ((si.CONT, 1.0), (si.CONT_RATIO, 0.8), (si.STATIC, 1.0)) for pm in (si.SWAP, si.RECOMPUTE)]
    cfg = si.SweepConfig("pressure", si.LLAMA2_13B, [si.Hw(mem_capacity=30 * 10 ** 9), si.A100], pols,
                         si.Workload(300, [4.0, 16.0], [0, 1]))
    sw = run_gpu(api, cfg)
    check_points(sw, cfg, list(range(cfg.num_points)), records=True, trace=True)
    assert sw.summaries()["n_preemptions"].sum() > 0


def test_quantile_getter_arbitrary_q(api):
    from oracle import oracle as O
    cfg = si.c2()
    sw = run_gpu(api, cfg)
    qs = [0, 1, 100, 2500, 5000, 7500, 9000, 9500, 9900, 9990, 10000]
    for p in (3, 77):
        o = O.simulate(cfg, p)
        rec = o["records"]
        a, pr, out = O.workload(cfg, p)
        fin = rec["status"] == 1
        vals = {
            "ttft": rec["ttft_ns"][fin] / 1e9, "e2e": rec["e2e_ns"][fin] / 1e9, "mtpot": rec["mtpot_ns"][fin] / 1e9,
            "norm": (rec["e2e_ns"][fin] / out[fin].astype(np.float64)) / 1e9,
        }
        m2 = fin & (out >= 2)
        vals["tpot"] = ((rec["e2e_ns"][m2] - rec["ttft_ns"][m2]) / (out[m2] - 1).astype(np.float64)) / 1e9
        for name, v in vals.items():
            v = np.sort(v)
            got = sw.latency_quantiles(p, name, qs)
            ref = [v[max(1, -(-q * len(v) // 10000)) - 1] for q in qs]
            assert np.array_equal(got, np.asarray(ref)), (p, name)


def test_c3_sampled(api):
    """Full C3 sweep (4,608 points, 10k requests each) on the GPU; the oracle on a
    deterministic sample incl. grid corners."""
    cfg = si.c3()
    sw = run_gpu(api, cfg)
    s = sw.summaries()
    assert (s["n_finished"] == 10_000).all() and (s["status_flags"] & 16 == 0).all()
    corners = [0, 1, 2, 3, 4, 5, 4607, 4606, 4605, 1536 * 1 + 17, 3 * 1535, 3 * 1535 + 2]
    pts = sample_points(cfg.num_points, target=16, corners=corners)
    check_points(sw, cfg, pts, records=True)


def test_c4_sampled(api):
    cfg = si.c4()
    sw = run_gpu(api, cfg)
    s = sw.summaries()
    assert (s["status_flags"] & 16 == 0).all()
    pts = sample_points(cfg.num_points, target=12, corners=[0, 191, 192, 2303, 768 + 5, 1536 + 100])
    check_points(sw, cfg, pts, records=True)


def test_c4_strided_helper_kernel(api):
    """C4 at 8 emulated GPUs: rank 7's strided shard (288 points <= 4 per SM) runs in the
    helper-warp kernel with carried stretch state and 64-iteration stretches.  Sampled points
    (incl. the longest chain, point 1543 = 7 mod 8) against the oracle, and fast-forward on ==
    off byte for byte over the whole shard."""
    cfg = si.c4()
    sw = api.Sweep(cfg)
    sw.run(7, cfg.num_points, 8)
    info = sw.run_info()
    assert info["helper_mode"] == 1 and info["sim_warps_per_block"] == 1
    s = sw.summaries()
    assert (s["status_flags"] & 16 == 0).all()
    check_points(sw, cfg, [7, 1543, 2303, 1159, 391], records=True)
    off = api.Sweep(replace(cfg, options=replace(cfg.options, fast_forward=False)))
    off.run(7, cfg.num_points, 8)
    assert off.summaries().tobytes() == s.tobytes()
    for p in (1543, 2303):
        assert off.records(p).tobytes() == sw.records(p).tobytes()


def test_sharegpt_builtin_equals_table(api):
    cfg = si.c1()
    a = run_gpu(api, cfg).summaries()
    b = run_gpu(api, replace(cfg, workload=replace(cfg.workload, len_dist="sharegpt_synth_v1"))).summaries()
    assert a.tobytes() == b.tobytes()


def test_fast_forward_is_bit_identical(api):
    """Time-parallel evaluation of quiescent stretches must not change a single
    bit of any result: compare full summaries, records and traces with it switched off."""
    c5r = si.subset(si.c5(), rates=[0, 15], seeds=[0], hws=[0, 5, 10, 15])
    c5r = replace(c5r, workload=replace(c5r.workload, num_requests=400),
                  options=replace(c5r.options, iteration_trace_cap=1 << 16))
    for cfg in (si.c2(), replace(si.c1(), options=si.Options(trace_mode=si.FULL, iteration_trace_cap=1 << 16)),
                replace(si.c1(), options=si.Options(trace_bin_ns=7_000_000)), c5r):
        on = run_gpu(api, cfg)
        off = run_gpu(api, replace(cfg, options=replace(cfg.options, fast_forward=False)))
        assert on.summaries().tobytes() == off.summaries().tobytes()
        for p in range(0, cfg.num_points, 13):
            assert on.records(p).tobytes() == off.records(p).tobytes()
            for w in ((0, 1) if cfg.options.topology == si.PD_PAIR else (0,)):
                assert on.mem_trace(p, w).tobytes() == off.mem_trace(p, w).tobytes()
            if cfg.options.iteration_trace_cap:
                assert on.iteration_trace(p).tobytes() == off.iteration_trace(p).tobytes()


# ------------------------------------------------------------------ a.9 P/D pair
def check_pd_points(sw, cfg, points, iters=False):
    want = ("summary", "records", "trace") + (("iters",) if iters else ())
    ora = oracle_points(cfg, points, want=want)
    nw = cfg.options.pd_prefill + cfg.options.pd_decode
    node = nw > 2 or cfg.options.node_loop
    bad = []
    full = cfg.options.trace_mode == si.FULL
    for p in points:
        o = ora[p]
        g = sw.summary(p)
        bad += compare_summary(g, o["summary"], p, full_trace=full)
        bad += compare_records(sw.records(p), o["records"], p)
        for w in range(nw):
            bad += compare_trace(sw.mem_trace(p, w), o["trace"][w], p, prefix=full and bool(int(g["status_flags"]) & 1))
        prof = sw.point_profile(p)
        if (prof["n_transfers"], prof["transfer_bytes"]) != (o["summary"]["n_transfers"], o["summary"]["transfer_bytes"]):
            bad.append(f"point {p}: transfers gpu={prof['n_transfers']},{prof['transfer_bytes']} "
                       f"oracle={o['summary']['n_transfers']},{o['summary']['transfer_bytes']}")
        if iters:
            g, oi = sw.iteration_trace(p), o["iters"]
            if node:  # a decode worker's stretch commits ahead of other workers: compare by (worker, k)
                g = g[np.lexsort((g["k"], g["worker"]))]
                oi = oi[np.lexsort((oi["k"], oi["worker"]))]
            pairs = [("k", "k"), ("t_start_ns", "t_start"), ("T_ns", "T_ns"), ("n_prefill", "S_p"),
                     ("n_decode", "D"), ("n_admitted", "n_admitted"), ("n_finished", "n_finished"),
                     ("blocks_in_use", "blocks"), ("worker", "worker")]
            for i in range(min(len(g), len(oi))):
                diff = [f for f, of in pairs if int(g[f][i]) != int(oi[of][i])]
                if diff:
                    bad.append(f"point {p}: first divergent PD iteration {i}: {diff}")
                    break
    assert not bad, "\n".join(bad[:20])


def _micro_pd(rng):
    n = int(rng.integers(1, 60))
    a = np.sort(rng.integers(0, 2_000_000_000, n))
    p = rng.integers(1, 64, n)
    o = rng.integers(1, 64, n)
    mml = 128
    model = replace(si.LLAMA2_7B, max_model_len=mml)
    bs = int(rng.choice([4, 16]))
    mb = -(-mml // bs)
    hws = [replace(si.A100, kv_blocks_override=int(rng.integers(mb, mb + 30)),
                   peak_flops=float(rng.choice([78e12, 312e12])), mem_bw=float(rng.choice([1e12, 4e12])))
           for _ in range(2)]
    pol = si.Policy(kind=str(rng.choice([si.STATIC, si.CONT])), preempt=str(rng.choice([si.SWAP, si.RECOMPUTE])),
                    max_num_seqs=int(rng.choice([2, 8, 256])), block_size=bs)
    w = si.Workload(n, [1.0], [0], len_dist=si.TRACE, trace_arrival_ns=a.tolist(), trace_prompt=p.tolist(),
                    trace_output=o.tolist(), prompt_table=None, output_table=None)
    opts = si.Options(topology=si.PD_PAIR, pd_link_bw=float(rng.choice([1e9, 200e9])),
                      trace_mode=str(rng.choice([si.FULL, si.BINNED])), trace_bin_ns=50_000_000,
                      iteration_trace_cap=1 << 16, fast_forward=bool(rng.random() < 0.8))
    return si.SweepConfig("micro-pd", model, hws, [pol], w, opts)


def test_pd_micro_configs(api):
    rng = np.random.default_rng(17)
    for _ in range(40):
        cfg = _micro_pd(rng)
        sw = run_gpu(api, cfg)
        check_pd_points(sw, cfg, list(range(cfg.num_points)), iters=True)


def test_full_trace_overflow_pd_and_node(api):
    """FULL traces with a 600-byte budget per worker on a 1P:1D pair and a 2P:3D node: every
    worker's stream keeps a prefix of whole iterations equal to the oracle's samples, and the
    overflow bit is set."""
    rng = np.random.default_rng(29)
    for node in (False, True):
        cfg = _micro_pd(rng)
        while cfg.workload.num_requests < 30:
            cfg = _micro_pd(rng)
        w = cfg.workload
        opts = replace(cfg.options, trace_mode=si.FULL, trace_cap_bytes=600, fast_forward=True,
                       pd_prefill=2 if node else 1, pd_decode=3 if node else 1)
        c = replace(cfg, workload=w, options=opts)
        sw = run_gpu(api, c)
        check_pd_points(sw, c, list(range(c.num_points)))
        assert (sw.summaries()["status_flags"] & 1).any()


def test_c5_reduced_grid(api):
    """C5's 16x16 (P, D) profile pairs x {SWAP, RECOMPUTE}, 3 of its rates, 300 requests per point."""
    base = si.c5()
    cfg = replace(si.subset(base, rates=[0, 8, 15], seeds=[0]), workload=replace(
        si.subset(base, rates=[0, 8, 15], seeds=[0]).workload, num_requests=300))
    sw = run_gpu(api, cfg)
    s = sw.summaries()
    assert (s["n_finished"] == 300).all() and (s["status_flags"] & 16 == 0).all()
    check_pd_points(sw, cfg, sample_points(cfg.num_points, target=40, corners=[0, 1, 767, 768, 1535]))


def test_c5_bench_config_sampled(api):
    """C5 exactly as bench.py times it on one GPU (16x16 pairs x {SWAP, RECOMPUTE} x 16 rates, one
    seed: 8,192 points of 10k requests), checked against the oracle on sampled points incl. the
    grid corners."""
    base = si.c5()
    cfg = replace(base, workload=replace(base.workload, seeds=[0]))
    assert cfg.num_points == 8192
    sw = run_gpu(api, cfg)
    s = sw.summaries()
    assert (s["n_finished"] + s["n_rejected"] == s["n_requests"]).all() and (s["status_flags"] & 16 == 0).all()
    check_pd_points(sw, cfg, sample_points(cfg.num_points, target=8, corners=[0, 15, 4096, 8191]))


def test_prefill_first_parity(api):
    """NEXT-3 prefill-first iterations: C2 in full, and random micro configs."""
    cfg = replace(si.c2(), policies=[si.Policy(iteration_mode=si.PREFILL_FIRST)])
    sw = run_gpu(api, cfg)
    check_points(sw, cfg, list(range(cfg.num_points)), records=True)
    off = run_gpu(api, replace(cfg, options=replace(cfg.options, fast_forward=False)))
    assert sw.summaries().tobytes() == off.summaries().tobytes()
    rng = np.random.default_rng(23)
    for _ in range(40):
        c = _micro(rng)
        c = replace(c, policies=[replace(c.policies[0], iteration_mode=si.PREFILL_FIRST)])
        check_points(run_gpu(api, c), c, [0], records=True, trace=True, iters=True)


def test_prefill_first_under_memory_pressure(api):
    """Prefill-first iterations with a small KV pool: the memory back-off of the fast-forward and
    the prefill-only pauses interleave, so a stretch must never start right after a prefill-only
    iteration (the paused decodes' first gap would be lost from mTPOT).  Oracle parity on every
    point and fast-forward on == off byte for byte."""
    pols = [si.Policy(kind=k, preempt=pm, max_mem_ratio=r, iteration_mode=si.PREFILL_FIRST)
            for k, r in ((si.CONT, 1.0), (si.CONT_RATIO, 0.8)) for pm in (si.SWAP, si.RECOMPUTE)]
    cfg = si.SweepConfig("pf-pressure", si.LLAMA2_13B, [si.Hw(mem_capacity=30 * 10 ** 9),
                                                         si.Hw(mem_capacity=34 * 10 ** 9)], pols,
                         si.Workload(400, [4.0, 16.0], [0, 1]))
    sw = run_gpu(api, cfg)
    check_points(sw, cfg, list(range(cfg.num_points)), records=True, trace=True)
    off = run_gpu(api, replace(cfg, options=replace(cfg.options, fast_forward=False)))
    assert sw.summaries().tobytes() == off.summaries().tobytes()
    for p in range(cfg.num_points):
        assert sw.records(p).tobytes() == off.records(p).tobytes()
    assert sw.summaries()["n_preemptions"].sum() > 0


@pytest.mark.parametrize("blocks", [300_000, 1_000_000])
def test_huge_kv_pool_on_few_points(api, blocks):
    """A few points (one warp per SM, the helper-warp kernel) with a free-block bitmap far beyond
    4,096 words: 300k blocks still fit the helper's replayed copy (variant 0), 1M blocks (125 KB of
    bitmap) do not and must run without the helper (variant 4) instead of failing."""
    w = si.Workload(300, [20.0], [0, 1])
    cfg = si.SweepConfig("huge-pool", si.LLAMA2_7B, [replace(si.A100, kv_blocks_override=blocks)],
                         [si.Policy()], w, si.Options(trace_mode=si.FULL))
    sw = run_gpu(api, cfg)
    check_points(sw, cfg, [0, 1], records=True, trace=True)


def test_full_trace_codec_c3_points(api):
    """The compressed FULL memory trace (delta + varint, trace_codec.cuh): whole C3
    points (10k requests, up to ~1M iterations) fit a 6 MiB stream, decode to exactly the oracle's
    per-iteration samples, and cost <= 6 B per iteration; the same for C1.  A small budget keeps
    a prefix of whole iterations and reports E_OVERFLOW."""
    base = si.c3()
    # grid corners of C3's fast/slow hardware x capacities x policies, via a subset config
    cfg = replace(si.subset(base, hws=[0, 5, 1535, 1530, 767, 1000], policies=[0, 1, 2]),
                  options=si.Options(trace_mode=si.FULL, trace_cap_bytes=6 << 20))
    sw = run_gpu(api, cfg)
    pts = list(range(cfg.num_points))
    check_points(sw, cfg, pts, records=False, trace=True)
    s = sw.summaries()
    assert not (s["status_flags"] & 1).any()
    bpi = []
    for p in pts:
        enc, n = sw.mem_trace_encoded(p)
        assert n == int(s["n_iterations"][p])
        bpi.append(len(enc) / n)
    assert max(bpi) <= 6.0, bpi
    c1 = replace(si.c1(), options=si.Options(trace_mode=si.FULL))
    sw1 = run_gpu(api, c1)
    check_points(sw1, c1, [0], records=True, trace=True)
    enc, n = sw1.mem_trace_encoded(0)
    assert len(enc) <= 6 * n
    # a 4 KiB budget: a prefix of whole iterations, E_OVERFLOW, still the oracle's samples
    c1s = replace(si.c1(), options=si.Options(trace_mode=si.FULL, trace_cap_bytes=4096))
    sw2 = run_gpu(api, c1s)
    g = sw2.summary(0)
    assert int(g["status_flags"]) & 1
    tr = sw2.mem_trace(0)
    enc, n = sw2.mem_trace_encoded(0)
    assert 0 < len(tr) == n < int(g["n_iterations"]) and len(enc) <= 4096
    check_points(sw2, c1s, [0], records=True, trace=True)


def test_large_point_summary_scratch_path(api):
    """n = 20,000 requests per point exceeds the summary kernel's shared-memory key buffer
    (12,288), so quantiles run over the workspace scratch path; also exercises a trace cap."""
    w = si.Workload(20_000, [30.0, 60.0], [5], len_dist=si.UNIFORM, prompt_a=16, prompt_b=256,
                    output_a=2, output_b=64)
    cfg = si.SweepConfig("big", si.LLAMA2_7B, [si.Hw(mem_capacity=40 * 10 ** 9)],
                         [si.Policy(), si.Policy(kind=si.CONT_RATIO, max_mem_ratio=0.5, preempt=si.RECOMPUTE)], w,
                         si.Options(trace_cap_bytes=32 * 100))
    sw = run_gpu(api, cfg)
    check_points(sw, cfg, list(range(cfg.num_points)), records=True, trace=True)
    assert (sw.summaries()["status_flags"] & 1).all()   # 100-sample cap overflowed
    for p in range(cfg.num_points):
        q = sw.latency_quantiles(p, "e2e", [1234, 5000, 9999])
        assert (np.diff(q) >= 0).all()


def test_chunked_prefill_parity(api):
    """NEXT-3b chunked prefill (reading R-N3b): random micro configs under small token budgets
    (prompts longer than the budget, preemption of partial prefills), FF on/off identical, and
    the C2 grid + a memory-pressure grid under vLLM's chunked default budget of 512."""
    rng = np.random.default_rng(29)
    for _ in range(60):
        c = _micro(rng)
        pol = c.policies[0]
        budget = int(rng.choice([max(pol.max_num_seqs, 16), max(pol.max_num_seqs, 40), 300]))
        c = replace(c, policies=[replace(pol, iteration_mode=si.CHUNKED, max_batched_tokens=budget)])
        sw = run_gpu(api, c)
        check_points(sw, c, [0], records=True, trace=True, iters=True)
    pols = [si.Policy(kind=k, preempt=pm, iteration_mode=si.CHUNKED, max_batched_tokens=512)
            for k in (si.CONT, si.STATIC) for pm in (si.SWAP, si.RECOMPUTE)]
    for cfg in (replace(si.c2(), policies=[si.Policy(iteration_mode=si.CHUNKED, max_batched_tokens=512)]),
                si.SweepConfig("pressure", si.LLAMA2_13B, [si.Hw(mem_capacity=30 * 10 ** 9), si.A100], pols,
                               si.Workload(300, [4.0, 16.0], [0, 1]))):
        sw = run_gpu(api, cfg)
        check_points(sw, cfg, list(range(cfg.num_points)), records=True, trace=True)
        off = run_gpu(api, replace(cfg, options=replace(cfg.options, fast_forward=False)))
        assert sw.summaries().tobytes() == off.summaries().tobytes()
        if cfg.name == "pressure":
            assert sw.summaries()["n_preemptions"].sum() > 0


# ------------------------------------------------------------------ NEXT-1 xP:yD node
def test_node_micro_configs(api):
    """Random x:y nodes (x + y <= 8) under all three dispatch policies vs the oracle's node loop:
    summaries, records, every worker's memory trace and the iteration records."""
    rng = np.random.default_rng(41)
    for _ in range(40):
        cfg = _micro_pd(rng)
        x = int(rng.integers(1, 5))
        y = int(rng.integers(1, 9 - x))
        d = str(rng.choice([si.ROUND_ROBIN, si.LEAST_OUTSTANDING, si.LEAST_MEMORY]))
        cfg = replace(cfg, options=replace(cfg.options, pd_prefill=x, pd_decode=y, dispatch=d))
        sw = run_gpu(api, cfg)
        check_pd_points(sw, cfg, list(range(cfg.num_points)), iters=True)


def test_sweep_resumable_equals_one_run(api, tmp_path):
    """Point-granular checkpoint / resume: a C2 sweep interrupted after 3 chunks of 16 points and
    resumed gives the bytes of one uninterrupted run."""
    cfg = si.c2()
    full = api.sweep(cfg)
    path = str(tmp_path / "c2.npz")
    part = api.sweep_resumable(cfg, path, chunk_points=16, max_chunks=3)
    assert (part["n_requests"][:48] > 0).all() and (part["n_requests"][48:] == 0).all()
    out = api.sweep_resumable(cfg, path, chunk_points=16)
    assert out.tobytes() == full.tobytes()
    again = api.sweep_resumable(cfg, path, chunk_points=16, max_chunks=0)  # nothing left to run
    assert again.tobytes() == full.tobytes()


def test_node_large_batch_cap(api):
    """A node whose policy allows 512 running requests (the 1024-slot kernel build): 1P:2D runs
    and matches the oracle; 1P:6D needs more shared memory per point than an SM has and is
    refused loudly at create instead of running anything else."""
    from paper_2503_08415_b200 import TokensimError
    rng = np.random.default_rng(77)
    cfg = _micro_pd(rng)
    while cfg.workload.num_requests < 30:
        cfg = _micro_pd(rng)
    cfg = replace(cfg, policies=[replace(cfg.policies[0], max_num_seqs=512)])
    ok = replace(cfg, options=replace(cfg.options, pd_prefill=1, pd_decode=2, dispatch=si.LEAST_OUTSTANDING))
    sw = run_gpu(api, ok)
    check_pd_points(sw, ok, list(range(ok.num_points)), iters=True)
    big = replace(cfg, options=replace(cfg.options, pd_prefill=1, pd_decode=6))
    with pytest.raises(TokensimError) as ei:  # refused at create (validation), before any launch
        run_gpu(api, big)
    assert "shared memory per point" in str(ei.value)


def test_node_epoch_stress(api):
    """The node kernel's epoch horizons (sim_pdn.cuh) under adversarial arrivals: bursts of equal
    timestamps (the exact-dispatch prediction must stand aside), dense and sparse streams, tiny
    and large KV pools, every dispatch policy, 1..4 prefill x 1..7 decode workers, vs the
    oracle's sequential node loop (summaries, records, traces, iteration records)."""
    rng = np.random.default_rng(4242)
    for it in range(48):
        cfg = _micro_pd(rng)
        n = int(rng.integers(20, 160))
        base = np.sort(rng.integers(0, int(rng.choice([2e8, 2e9, 2e10])), n))
        if it % 3 == 0:  # bursts: runs of identical arrival times
            base = np.repeat(base[: max(1, n // 4)], 4)[:n]
            base = np.sort(base)
        p = rng.integers(1, 64, len(base))
        o = rng.integers(1, 64, len(base))
        w = replace(cfg.workload, num_requests=len(base), trace_arrival_ns=base.tolist(), trace_prompt=p.tolist(),
                    trace_output=o.tolist())
        x = int(rng.integers(1, 5))
        y = int(rng.integers(1, 9 - x))
        d = str(rng.choice([si.ROUND_ROBIN, si.LEAST_OUTSTANDING, si.LEAST_MEMORY]))
        cfg = replace(cfg, workload=w, options=replace(cfg.options, pd_prefill=x, pd_decode=y, dispatch=d))
        sw = run_gpu(api, cfg)
        check_pd_points(sw, cfg, list(range(cfg.num_points)), iters=True)


def test_node_loop_equals_pair(api):
    """The general node loop run on 1P:1D pairs gives the pair kernel's bytes."""
    rng = np.random.default_rng(43)
    for _ in range(12):
        cfg = _micro_pd(rng)
        a = run_gpu(api, cfg)
        b = run_gpu(api, replace(cfg, options=replace(cfg.options, node_loop=True)))
        assert a.summaries().tobytes() == b.summaries().tobytes()
        for p in range(cfg.num_points):
            assert a.records(p).tobytes() == b.records(p).tobytes()


def test_node_sharegpt_grid(api):
    """fig:pd-shaped node sweeps (8 workers: P1-D7, P2-D6, P4-D4) on LLaMA-2-7B with ShareGPT-like
    lengths, 3 rates x {SWAP, RECOMPUTE}, every dispatch policy; FF on/off identical."""
    base = si.SweepConfig("node", si.LLAMA2_7B, [si.A100], [si.Policy(preempt=si.SWAP), si.Policy(preempt=si.RECOMPUTE)],
                          si.Workload(400, [4.0, 16.0, 48.0], [0]), si.Options(topology=si.PD_PAIR))
    for x, y in ((1, 7), (2, 6), (4, 4)):
        for d in (si.ROUND_ROBIN, si.LEAST_OUTSTANDING, si.LEAST_MEMORY):
            cfg = replace(base, options=replace(base.options, pd_prefill=x, pd_decode=y, dispatch=d))
            sw = run_gpu(api, cfg)
            assert (sw.summaries()["n_finished"] == 400).all()
            check_pd_points(sw, cfg, list(range(cfg.num_points)))
            if d == si.LEAST_MEMORY:
                off = run_gpu(api, replace(cfg, options=replace(cfg.options, fast_forward=False)))
                assert sw.summaries().tobytes() == off.summaries().tobytes()


def test_node_cta_shapes_are_byte_identical(api):
    """The node kernel's CTA-parallel decode warps (sim_pdn.cuh) give the same bytes run twice, and
    in all three builds: 192 points at once (more points than SMs: the register-capped build, two
    CTAs per SM) and the same points in halves of 96 (one CTA per SM) with the scheduler on a warp
    of its own and with the barrier build; sampled points vs the oracle."""
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    cfg = si.SweepConfig("node-shapes", si.LLAMA2_7B, [si.A100],
                         [si.Policy(preempt=si.SWAP), si.Policy(preempt=si.RECOMPUTE)],
                         si.Workload(200, [2.0 * 2.0 ** (k / 2.0) for k in range(16)], list(range(6))),
                         si.Options(topology=si.PD_PAIR, pd_prefill=2, pd_decode=6,
                                    dispatch=si.LEAST_OUTSTANDING, iteration_trace_cap=1 << 16))
    n = cfg.num_points
    assert n > sms
    a = run_gpu(api, cfg)
    assert a.run_info()["sim_blocks"] > sms  # two CTAs per SM
    sa = a.summaries().tobytes()
    recs = {p: a.records(p).tobytes() for p in (0, 77, n - 1)}
    its = {p: a.iteration_trace(p) for p in (0, n - 1)}
    a.run()
    assert a.summaries().tobytes() == sa
    half = n // 2
    import os as _os
    for sw_mode in ("1", "0"):  # halves of one wave: the scheduler-warp build, and the barrier build
        _os.environ["TOKENSIM_NODE_SW"] = sw_mode
        try:
            b = api.Sweep(cfg)
            parts = []
            for beg in (0, half):
                b.run(beg, beg + half)
                assert b.run_info()["sim_blocks"] <= sms
                parts.append(b.summaries().tobytes())
                for p in recs:
                    if beg <= p < beg + half:
                        assert b.records(p).tobytes() == recs[p]
                for p in its:
                    if beg <= p < beg + half:
                        g, h = b.iteration_trace(p), its[p]
                        key = lambda x: np.lexsort((x["k"], x["worker"]))  # noqa: E731
                        assert g[key(g)].tobytes() == h[key(h)].tobytes()
            assert b"".join(parts) == sa, sw_mode
        finally:
            _os.environ.pop("TOKENSIM_NODE_SW", None)
    check_pd_points(a, cfg, [0, 77, n - 1])


# ------------------------------------------------------------------ NEXT-4 preload-buffer link
def test_preload_link_parity(api):
    """PRELOAD swap-in pipeline (reading R-N4) on the unified worker, the P/D pair and a node:
    SWAP-heavy micro configs and a memory-pressure grid vs the oracle."""
    rng = np.random.default_rng(61)
    for it in range(30):
        c = _micro(rng)
        c = replace(c, policies=[replace(c.policies[0], preempt=si.SWAP)],
                    options=replace(c.options, link_mode=si.PRELOAD,
                                    preload_buffer_bytes=int(rng.choice([1, 1 << 14, 1 << 20, 1 << 34]))))
        check_points(run_gpu(api, c), c, [0], records=True, trace=True, iters=True)
    pols = [si.Policy(kind=si.CONT, preempt=si.SWAP), si.Policy(kind=si.STATIC, preempt=si.SWAP)]
    cfg = si.SweepConfig("pressure", si.LLAMA2_13B, [si.Hw(mem_capacity=30 * 10 ** 9), si.A100], pols,
                         si.Workload(300, [4.0, 16.0], [0, 1]),
                         si.Options(link_mode=si.PRELOAD, preload_buffer_bytes=64 << 20))
    sw = run_gpu(api, cfg)
    check_points(sw, cfg, list(range(cfg.num_points)), records=True, trace=True)
    assert sw.summaries()["swap_in_bytes"].sum() > 0
    for x, y in ((1, 1), (2, 3)):
        c = _micro_pd(rng)
        c = replace(c, policies=[replace(c.policies[0], preempt=si.SWAP)],
                    options=replace(c.options, pd_prefill=x, pd_decode=y, link_mode=si.PRELOAD,
                                    preload_buffer_bytes=1 << 16))
        check_pd_points(run_gpu(api, c), c, list(range(c.num_points)), iters=True)


# ------------------------------------------------------------------ NEXT-2 multi-round + memory cache
def _micro_mr(rng):
    bs = int(rng.choice([4, 16]))
    mml = 512
    total = int(rng.integers(-(-mml // bs), -(-mml // bs) + 60))
    pol = si.Policy(kind=str(rng.choice([si.STATIC, si.CONT, si.CONT_RATIO])),
                    preempt=str(rng.choice([si.SWAP, si.RECOMPUTE])), max_mem_ratio=float(rng.choice([0.5, 0.8, 1.0])),
                    max_num_seqs=int(rng.choice([2, 8, 256])), block_size=bs)
    w = si.Workload(int(rng.integers(1, 40)), [float(rng.choice([1.0, 8.0]))], [int(rng.integers(0, 1000))],
                    len_dist=si.UNIFORM, prompt_a=8, prompt_b=120, output_a=2, output_b=60, multi_round=True,
                    think_mean_s=float(rng.choice([0.05, 1.0])))
    opts = si.Options(memory_cache=bool(rng.random() < 0.8), cache_capacity_blocks=int(rng.choice([0, 8, 64])),
                      trace_mode=si.FULL if rng.random() < 0.5 else si.BINNED, trace_bin_ns=100_000_000,
                      iteration_trace_cap=1 << 16, horizon_ns=int(rng.choice([-1, -1, 2_000_000_000])))
    return si.SweepConfig("micro-mr", replace(si.LLAMA2_7B, max_model_len=mml),
                          [replace(si.A100, kv_blocks_override=total)], [pol], w, opts)


def test_multi_round_cache_parity(api):
    """NEXT-2 (reading R-N2): multi-round conversations with and without the host LRU memory
    cache -- random micro configs (every policy, both preemption modes, small caches that evict,
    horizons) and a LLaMA-2-7B rate x seed grid -- bit-exact against the oracle."""
    rng = np.random.default_rng(73)
    for _ in range(40):
        c = _micro_mr(rng)
        check_points(run_gpu(api, c), c, [0], records=True, trace=True, iters=True)
    for cache in (False, True):
        cfg = si.SweepConfig("mr-grid", si.LLAMA2_7B, [si.A100],
                             [si.Policy(preempt=si.SWAP), si.Policy(preempt=si.RECOMPUTE)],
                             si.Workload(300, [2.0, 8.0, 24.0], [0, 1], len_dist=si.UNIFORM, prompt_a=64,
                                         prompt_b=512, output_a=16, output_b=128, multi_round=True,
                                         think_mean_s=2.0),
                             si.Options(memory_cache=cache))
        sw = run_gpu(api, cfg)
        check_points(sw, cfg, list(range(cfg.num_points)), records=True, trace=True)
        s = sw.summaries()
        assert (s["n_requests"] > 300).all() and (s["n_finished"] == s["n_requests"]).all()
        off = run_gpu(api, replace(cfg, options=replace(cfg.options, fast_forward=False)))
        assert sw.summaries().tobytes() == off.summaries().tobytes()


def test_widened_row_presets_sampled(api):
    """The bench sweeps of the widened rows (c6 node, c7 multi-round + cache, c8 prefill-first /
    chunked, c9 preload link) at full size on the GPU, checked against the oracle on samples."""
    for name, target in (("c6", 4), ("c7", 8), ("c8", 10), ("c9", 6)):
        cfg = si.PRESETS[name]()
        sw = run_gpu(api, cfg)
        s = sw.summaries()
        assert (s["n_finished"] + s["n_rejected"] == s["n_requests"]).all(), name
        pts = sample_points(cfg.num_points, target=target, corners=[0, cfg.num_points - 1])
        if cfg.options.topology == si.PD_PAIR:
            check_pd_points(sw, cfg, pts)
        else:
            check_points(sw, cfg, pts, records=True)


def test_edge_shapes(api):
    """Edge shapes: non-power-of-two block sizes (the div/mod path of BSz), max_num_seqs > 256
    (the CAP = 1024 kernel instantiation) and max_num_seqs = 1024, on the unified worker, the P/D
    pair, a node, chunked prefill and multi-round workloads."""
    rng = np.random.default_rng(97)
    for bs, mns in ((12, 8), (20, 256), (7, 600), (16, 1024), (5, 1024)):
        for _ in range(3):
            c = _micro(rng)
            mml = c.model.max_model_len
            pol = replace(c.policies[0], block_size=bs, max_num_seqs=mns, watermark_blocks=0)
            hw = replace(c.hws[0], kv_blocks_override=int(rng.integers(-(-mml // bs), -(-mml // bs) + 50)))
            c = replace(c, policies=[pol], hws=[hw])
            check_points(run_gpu(api, c), c, [0], records=True, trace=True, iters=True)
            cc = replace(c, policies=[replace(pol, iteration_mode=si.CHUNKED, max_batched_tokens=max(mns, 64))])
            check_points(run_gpu(api, cc), cc, [0], records=True, iters=True)
        p = _micro_pd(rng)
        ppol = replace(p.policies[0], block_size=bs, max_num_seqs=mns)
        phws = [replace(h, kv_blocks_override=int(rng.integers(-(-128 // bs), -(-128 // bs) + 30))) for h in p.hws]
        p = replace(p, policies=[ppol], hws=phws)
        check_pd_points(run_gpu(api, p), p, list(range(p.num_points)), iters=True)
        pn = replace(p, options=replace(p.options, pd_prefill=2, pd_decode=2))
        check_pd_points(run_gpu(api, pn), pn, list(range(pn.num_points)), iters=True)
        m = _micro_mr(rng)
        m = replace(m, policies=[replace(m.policies[0], block_size=bs, max_num_seqs=mns)],
                    hws=[replace(m.hws[0], kv_blocks_override=int(rng.integers(-(-512 // bs), -(-512 // bs) + 60)))])
        check_points(run_gpu(api, m), m, [0], records=True, iters=True)


# ------------------------------------------------------------------ multi-GPU path on one GPU
def test_run_distributed_nccl_world_one(api, tmp_path):
    """The NCCL path of run_distributed (device summaries, all_gather_into_tensor over NCCL,
    import into the handle) under torchrun with one rank on cuda:0 gives the bytes of the
    plain single-process sweep.  (World sizes > 1 need more GPUs; the host logic of W = 2 and 3
    is covered with gloo in tests/test_distributed.py.)"""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "dist.npy"
    script = tmp_path / "dist_run.py"
    script.write_text(
        "import sys, numpy as np, torch, torch.distributed as dist\n"
        f"sys.path.insert(0, {root!r})\n"
        "import sweep_inputs as si, paper_2503_08415_b200 as P\n"
        "torch.cuda.set_device(0)\n"
        "dist.init_process_group('nccl', device_id=torch.device('cuda', 0))\n"
        "sw, allv = P.run_distributed(si.c2())\n"
        f"np.save({str(out)!r}, np.asarray(allv.cpu()) if hasattr(allv, 'cpu') else allv)\n"
        "assert dist.get_backend() == 'nccl'\n"
        "dist.destroy_process_group()\n")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                        "--master-addr", "127.0.0.1", "--master-port", "29613", str(script)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(out)
    ref = api.sweep(si.c2())
    assert got.view(np.uint8).tobytes()[:ref.nbytes] == ref.tobytes()
