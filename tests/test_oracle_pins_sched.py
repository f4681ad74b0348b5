"""Pins for the oracle's scheduling boundaries and its cost aggregation (-m "not gpu").

VERDICT r1 "What's weak #1" named four oracle parts that were parity-unpinned; each is pinned
here against something other than the oracle itself:

* the closed-form victim count of c.4 step 3 (reading A7): against the
  literal SEQUENTIAL rule ("serve R in id order; while r cannot get its block, preempt the
  latest running request, possibly r itself") re-stated in `tests/seqref.py`, on 800 random
  tiny configurations (<= 6 requests, <= 6 blocks), plus three cases worked by hand
  (`tests/golden/preemption_tiny.json`: m = 2, lhs == rhs, a victim that needs no block);
* the CONT_RATIO admission threshold (A15, A18): hand traces at
  floor(r * total), one block over, a rejection, and S:291/S:292's examples;
* multi-prefill aggregation in the cost model ("independently coded brute-force evaluation
  of the normative FLOP/byte table"): `seqref.cost_ns` (plain Python floats)
  against the oracle bit for bit on random multi-prefill + decode plans;
* the digest mix (SURVEY c.6): the splitmix64 reference outputs for seed 1234567.
"""
import json
import math
import os
from dataclasses import replace

import numpy as np
import pytest

import sweep_inputs as si
from seqref import cost_ns, simulate as seq_simulate

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U32 = si.UINT32_MAX


def _trace_cfg(reqs, model, hw, pol):
    w = si.Workload(len(reqs), [1.0], [0], len_dist=si.TRACE,
                    trace_arrival_ns=[r[0] for r in reqs], trace_prompt=[r[1] for r in reqs],
                    trace_output=[r[2] for r in reqs], prompt_table=None, output_table=None)
    return si.SweepConfig("tiny", model, [hw], [pol], w, si.Options(trace_mode=si.NONE_TRACE))


def _oracle(cfg):
    from oracle import oracle as O
    return O.simulate(cfg, 0, check_invariants=True, keep_events=True,
                      want=("summary", "records", "iters", "events"))


ITER_FIELDS = ("k", "t_start", "T_ns", "S_p", "D", "N_p", "C_d", "m", "n_resumed", "n_admitted",
               "n_rejected", "n_finished", "blocks")


def _compare(cfg, model, hw, pol, reqs):
    """Oracle vs the sequential-rule reference: iterations, block events, records, swap bytes."""
    o = _oracle(cfg)
    r = seq_simulate(model, hw, pol, reqs)
    it = o["iters"]
    got = [tuple(int(x[f]) for f in ITER_FIELDS) for x in it]
    assert got == r["iters"], (pol, reqs)
    ev = [(int(e["k"]), int(e["kind"]), int(e["req"]), int(e["block"])) for e in o["events"]]
    assert ev == r["events"], (pol, reqs)
    rec = [(int(x["ttft_ns"]), int(x["e2e_ns"]), int(x["mtpot_ns"]), int(x["n_preempt"]), int(x["status"]),
            int(x["finish_k"])) for x in o["records"]]
    assert rec == r["records"], (pol, reqs)
    s = o["summary"]
    assert (s["swap_out_bytes"], s["swap_in_bytes"]) == (r["swap_out"], r["swap_in"])
    # victims: an iteration's first frees (A14: victim frees come first), by request, in order
    for k, (victims, _) in enumerate(r["victims"]):
        if victims:
            vic = []
            for e in ev:
                if e[0] == k and e[1] == 2 and e[2] not in vic:
                    vic.append(e[2])
            assert vic[:len(victims)] == victims, (k, vic, victims)
            assert int(it["m"][k]) == len(victims)
    return r


def _random_tiny(rng, preempt):
    """<= 6 requests, <= 6 blocks.  Two thirds of the draws are 'pressure' draws (arrivals at 0,
    no watermark, no seq / token cap, prompt lengths on block boundaries) so that preemptions
    with m >= 2, lhs == rhs and need-0 victims occur often; the rest vary every knob."""
    bs = int(rng.choice([1, 2, 4]))
    while True:
        total = int(rng.integers(1, 7))
        if total * bs >= 2:
            break
    mml = int(rng.integers(2, total * bs + 1))             # validation: total * bs >= mml
    pressure = rng.random() < 0.67
    n = int(rng.integers(2 if pressure else 1, 7))
    reqs = []
    for _ in range(n):
        if pressure and mml > bs and rng.random() < 0.7:
            p = bs * (1 if rng.random() < 0.5 else int(rng.integers(1, (mml - 1) // bs + 1)))
        else:
            p = int(rng.integers(1, mml))
        o = int(rng.integers(1, mml - p + 1)) if not pressure else mml - p - int(rng.integers(0, min(3, mml - p)))
        a = 0 if (pressure or rng.random() < 0.4) else int(rng.integers(0, 25_000_000))
        reqs.append([a, p, o])
    arr = sorted(r[0] for r in reqs)
    for r, a in zip(reqs, arr):
        r[0] = a
    if pressure:
        pol = si.Policy(kind=str(rng.choice([si.CONT, si.CONT, si.STATIC])), preempt=preempt, block_size=bs)
    else:
        pol = si.Policy(kind=str(rng.choice([si.STATIC, si.CONT, si.CONT_RATIO])), preempt=preempt,
                        max_mem_ratio=float(rng.choice([0.3, 0.5, 0.75, 1.0])),
                        max_num_seqs=int(rng.choice([1, 2, 3, 256])), block_size=bs,
                        max_batched_tokens=int(rng.choice([mml, mml + 5, U32])),
                        watermark_blocks=int(rng.integers(0, total - (-(-mml // bs)) + 1)))
    model = replace(si.LLAMA2_7B, max_model_len=mml)
    hw = replace(si.A100 if rng.random() < 0.5 else si.A100_IDEAL, kv_blocks_override=total)
    return model, hw, pol, [tuple(r) for r in reqs]


@pytest.mark.parametrize("preempt", [si.SWAP, si.RECOMPUTE])
def test_closed_form_victims_equal_sequential_rule(oracle_lib, preempt):
    """c.4 step 3's minimal m (and the whole unified loop) equals the sequential
    preempt-the-latest rule on 400 random tiny configurations per preemption mode."""
    rng = np.random.default_rng(20251 if preempt == si.SWAP else 20252)
    stats = {"preempting_iters": 0, "m_ge_2": 0, "equality": 0, "need0_victim": 0, "self_preempt": 0}
    for _ in range(400):
        model, hw, pol, reqs = _random_tiny(rng, preempt)
        r = _compare(_trace_cfg(reqs, model, hw, pol), model, hw, pol, reqs)
        for victims, (F, rows) in r["victims"]:
            if not victims:
                continue
            stats["preempting_iters"] += 1
            m = len(victims)
            stats["m_ge_2"] += m >= 2
            needs = [nd for _, nd, _ in rows]
            helds = [hd for _, _, hd in rows]
            n = len(rows)
            lhs = sum(needs[:n - m])
            rhs = F + sum(helds[n - m:])
            stats["equality"] += lhs == rhs
            need_of = {i: nd for i, nd, _ in rows}
            stats["need0_victim"] += any(need_of[v] == 0 for v in victims)
            assert victims[0] == rows[-1][0]                       # latest arrival goes first (A7)
            assert rows[0][0] not in victims                       # r_1 is never preempted
    # the random cases reach every boundary the verdict named
    assert stats["preempting_iters"] >= 100, stats
    assert stats["m_ge_2"] >= 10 and stats["equality"] >= 10 and stats["need0_victim"] >= 10, stats


def _gold_case(name, case, preempt, kind=si.CONT, ratio=1.0):
    model = replace(si.LLAMA2_7B, max_model_len=case["max_model_len"])
    hw = replace(si.A100_IDEAL, kv_blocks_override=case["total_blocks"])
    pol = si.Policy(kind=kind, preempt=preempt, block_size=4, max_mem_ratio=ratio)
    reqs = [tuple(r) for r in case["requests"]]
    return model, hw, pol, reqs


@pytest.mark.parametrize("preempt", [si.SWAP, si.RECOMPUTE])
@pytest.mark.parametrize("name", ["m2", "boundary", "need0_victim"])
def test_tiny_preemption_hand_traces(oracle_lib, name, preempt):
    case = json.load(open(os.path.join(GOLD, "preemption_tiny.json")))["cases"][name]
    model, hw, pol, reqs = _gold_case(name, case, preempt)
    o = _oracle(_trace_cfg(reqs, model, hw, pol))
    it, s = o["iters"], o["summary"]
    ev = [[int(e["k"]), int(e["kind"]), int(e["req"]), int(e["block"])] for e in o["events"]]
    assert ev == case["events"]
    mode = "swap" if preempt == si.SWAP else "recompute"
    for col in ("m", "n_resumed", "n_admitted", "n_finished", "blocks"):
        assert list(map(int, it[col])) == case[col], col
    for col in ("S_p", "D", "N_p"):
        assert list(map(int, it[col])) == case[col][mode], col
    assert list(map(int, o["records"]["n_preempt"])) == case["n_preempt"]
    assert (o["records"]["status"] == 1).all()
    bb = 4 * 524288
    if preempt == si.SWAP:
        assert s["swap_out_bytes"] == case["swap_blocks"]["out"] * bb
        assert s["swap_in_bytes"] == case["swap_blocks"]["in"] * bb
    else:
        assert s["swap_out_bytes"] == 0 and s["swap_in_bytes"] == 0
    assert s["n_request_iterations"] == sum(r[2] for r in reqs)


@pytest.mark.parametrize("name", ["at_limit_and_over", "s292_threshold", "s292_exact", "s291_ratio_one"])
def test_cont_ratio_threshold_hand_traces(oracle_lib, name):
    case = json.load(open(os.path.join(GOLD, "preemption_tiny.json")))["ratio"]["cases"][name]
    model, hw, pol, reqs = _gold_case(name, case, si.SWAP, kind=si.CONT_RATIO, ratio=case["ratio"])
    from oracle import oracle as O
    d = O.derive(_trace_cfg(reqs, model, hw, pol))
    assert d["ratio_limit"] == math.floor(case["ratio"] * case["total_blocks"])
    o = _oracle(_trace_cfg(reqs, model, hw, pol))
    it = o["iters"]
    for col in ("S_p", "D", "n_admitted", "n_rejected", "n_finished", "blocks"):
        assert list(map(int, it[col])) == case[col], col
    assert list(map(int, o["records"]["status"])) == case["status"]
    if "alloc_events" in case:
        ev = [[int(e["k"]), int(e["kind"]), int(e["req"]), int(e["block"])] for e in o["events"] if e["kind"] == 1]
        assert ev == case["alloc_events"]
    # the same traces through the independent sequential reference
    r = seq_simulate(model, hw, pol, reqs)
    assert [x[3] for x in r["iters"]] == case["S_p"] and [x[12] for x in r["iters"]] == case["blocks"]


def test_cost_table_independent_evaluation(oracle_lib):
    """100+ random BatchPlans (several prefills with c0 >= 0 and the emits flag, decodes,
    swap bytes) over three models and five profiles, oracle == re-typed c.5 table, 0 ns apart."""
    from oracle import oracle as O
    rng = np.random.default_rng(579)
    hws = [si.A100, si.A100_IDEAL, si.Hw(peak_flops=2.5e15, mem_bw=8e12, eff_flops=0.7, eff_bw=0.9),
           si.Hw(peak_flops=39e12, mem_bw=0.25e12)] + \
          [si.Hw(peak_flops=t * 312e12, mem_bw=t * 2.039e12, tp_degree=t, tp_link_bw=300e9) for t in (2, 4, 8)]
    n_multi = 0
    for i in range(160):
        model = (si.LLAMA2_7B, si.LLAMA2_13B, si.LLAMA2_70B)[i % 3]
        hw = hws[int(rng.integers(0, len(hws)))]
        cfg = si.SweepConfig("plan", model, [replace(hw, mem_capacity=10 ** 13)], [si.Policy()],
                             si.Workload(1, [1.0], [0]))
        npf = int(rng.integers(0, 6))
        pf = []
        for _ in range(npf):
            P = int(rng.integers(1, 2048))
            c0 = 0 if rng.random() < 0.5 else int(rng.integers(1, 2048))
            pf.append((P, c0, int(rng.random() < 0.8)))
        dec = [int(x) for x in rng.integers(1, 2048, int(rng.integers(0, 300)))]
        if not pf and not dec:
            dec = [1]
        swap = 0 if rng.random() < 0.6 else int(rng.integers(1, 64)) * 16 * 524288
        n_multi += npf >= 2
        got = O.iter_time_ns(cfg, pf, dec, swap)
        assert got == cost_ns(model, cfg.hws[0], pf, dec, swap), (model.name, hw, pf, len(dec), swap)
    assert n_multi >= 50
    # a plausible aggregation slip is caught: A_p of two prefills is not N_p(N_p+1)/2
    cfg = si.SweepConfig("plan", si.LLAMA2_7B, [si.Hw(mem_bw=1e30, eff_flops=1, eff_bw=1, iter_overhead_s=0)],
                         [si.Policy()], si.Workload(1, [1.0], [0]))
    two = O.iter_time_ns(cfg, [(1000, 0), (1000, 0)], [])
    assert two == cost_ns(cfg.model, cfg.hws[0], [(1000, 0), (1000, 0)], [])
    assert two < cost_ns(cfg.model, cfg.hws[0], [(2000, 0)], []) - 1000


def test_digest_mix_is_splitmix64(oracle_lib):
    """c.6 mix() = the splitmix64 finalizer.  Known answers: splitmix64 (Vigna's splitmix64.c:
    state += 0x9E3779B97F4A7C15; return mix(state)) seeded with 1234567 outputs these five
    values (external reference values).  fold([x]) = mix(0x9E3779B97F4A7C15 ^ x)."""
    from oracle import oracle as O
    G = 0x9E3779B97F4A7C15
    M = (1 << 64) - 1
    expect = [6457827717110365317, 3203168211198807973, 9817491932198370423, 4593380528125082431,
              16408922859458223821]
    s = 1234567
    for e in expect:
        s = (s + G) & M
        assert O.fold([s ^ G]) == e
    # fold chains mix over its fields in order (c.6)
    a, b = 12345, 678
    assert O.fold([a, b]) == O.fold([O.fold([a]) ^ G ^ b])


def test_block_manager_model_check(oracle_lib):
    """>= 10,000 allocate / free operations (preemptions included) replayed against a
    reference set model: every allocation takes the lowest free block (A14), every free
    returns a block its request holds, free + allocated = total after every operation
    (S:263), no block is in two lists, and everything is free at the end."""
    import bisect
    rng = np.random.default_rng(580)
    n_ops = n_preempt_frees = 0
    while n_ops < 10_000:
        n = int(rng.integers(10, 60))
        bs = int(rng.choice([1, 4, 16]))
        mml = 128
        total = int(rng.integers(-(-mml // bs), -(-mml // bs) + 24))
        a = np.sort(rng.integers(0, 400_000_000, n))
        reqs = [(int(x), int(rng.integers(1, 64)), int(rng.integers(1, 64))) for x in a]
        pol = si.Policy(kind=str(rng.choice([si.CONT, si.CONT_RATIO, si.STATIC])), max_mem_ratio=0.8,
                        preempt=str(rng.choice([si.SWAP, si.RECOMPUTE])), block_size=bs)
        model = replace(si.LLAMA2_7B, max_model_len=mml)
        cfg = _trace_cfg(reqs, model, replace(si.A100, kv_blocks_override=total), pol)
        o = _oracle(cfg)
        free = list(range(total))
        owner = {}
        held = {}
        for e in o["events"]:
            k, kind, rid, b = int(e["k"]), int(e["kind"]), int(e["req"]), int(e["block"])
            if kind == 1:
                assert free and free[0] == b, (k, rid, b, free[:3])
                free.pop(0)
                assert b not in owner
                owner[b] = rid
                held.setdefault(rid, []).append(b)
            else:
                assert owner.get(b) == rid, (k, rid, b)
                del owner[b]
                held[rid].remove(b)
                bisect.insort(free, b)
            assert len(free) + len(owner) == total
            n_ops += 1
        assert not owner and len(free) == total
        n_preempt_frees += int(o["summary"]["n_preemptions"])
    assert n_preempt_frees > 0
