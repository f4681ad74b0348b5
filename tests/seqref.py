"""An independent, literal pure-Python re-statement of the unified worker loop for TINY inputs.

TEST INFRASTRUCTURE ONLY.  It exists to pin the C++ oracle (oracle/oracle.cpp) against
something other than itself, as VERDICT r1 "Next round #1" asks.  It imports nothing from
oracle/ or from the product package and shares no code with either: the cost model below is
re-typed from SURVEY §8(c.5) in plain Python floats (IEEE binary64, the same rounding as C
doubles), and the loop is SURVEY §8(c.4) with ONE deliberate difference:

* Decode reservation uses the SEQUENTIAL preemption rule that SURVEY c.4 step 3 claims the
  closed form equals (reading A7; vLLM's `_schedule_running`): serve
  the running requests in arrival (id) order; while the request being served needs a block and
  none is free, preempt the latest-arrived request still running -- possibly the request
  itself.  The oracle instead computes the minimal victim count m in closed form.  Equal victim
  sets on every iteration of many random tiny configurations pin that closed form (including
  its boundary lhs == rhs and victims that need no block).

Physical block ids follow reading A14 (victim frees -> decode allocations in id order ->
resumes -> fresh admissions -> commit frees, lowest free index first, frees in logical order),
so events can be compared one for one.

Only what the tiny pins need is here: TRACE workloads (explicit arrays), MIXED iterations,
STATIC / CONT / CONT_RATIO, SWAP / RECOMPUTE, max_num_seqs, max_batched_tokens, watermark,
kv_blocks_override capacities.  Pure-Python loops: small cases only.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Tuple


# ----------------------------------------------------------------------------- c.5 cost model
def cost_ns(model, hw, prefills, decodes, swap_bytes: int = 0) -> int:
    """T_ns of one iteration, re-typed from SURVEY §8(c.5) (table + normative fp64 order).

    prefills: [(P, c0) or (P, c0, emits)]; decodes: [c_i = ctx_i + 1].  Every F_o / B_o is an
    exact Python int; float() rounds it to nearest like the C (double)u64 conversion."""
    s = model.dtype_bytes
    L = model.num_layers
    h = model.hidden
    q = model.num_heads * model.head_dim
    g = model.num_kv_heads * model.head_dim
    f = model.ffn_dim
    fu = 2 * f if model.gated_mlp else f
    V = model.vocab
    invF = 1.0 / (hw.peak_flops * hw.eff_flops)   # product first, then the division (c.1)
    invB = 1.0 / (hw.mem_bw * hw.eff_bw)
    invH = 1.0 / hw.host_link_bw
    Np = Ap = Kp = Sp = 0
    for e in prefills:
        P, c0 = int(e[0]), int(e[1])
        emits = bool(e[2]) if len(e) > 2 else True
        Np += P
        Ap += P * c0 + P * (P + 1) // 2          # causal: token j of the entry sees c0 + j keys
        Kp += c0 + P
        Sp += 1 if emits else 0
    D = len(decodes)
    Cd = sum(int(c) for c in decodes)
    N = Np + D
    S = Sp + D

    def roof(F: int, B: int) -> float:
        a = float(F) * invF
        b = float(B) * invB
        return a if a >= b else b

    t_qkv = roof(2 * N * h * (q + 2 * g), s * (h * (q + 2 * g) + N * h + N * (q + 2 * g))) if N > 0 else 0.0
    t_attp = roof(4 * q * Ap, s * (Np * (2 * q + 2 * g) + 2 * g * Kp)) if Np > 0 else 0.0
    t_attd = roof(4 * q * Cd, s * (D * (2 * q + 2 * g) + 2 * g * Cd)) if D > 0 else 0.0
    t_o = roof(2 * N * q * h, s * (q * h + N * q + N * h)) if N > 0 else 0.0
    t_up = roof(2 * N * h * fu, s * (h * fu + N * h + N * fu)) if N > 0 else 0.0
    t_down = roof(2 * N * f * h, s * (f * h + N * f + N * h)) if N > 0 else 0.0
    t_lm = roof(2 * S * h * V, s * (V * h + S * h + S * V)) if S > 0 else 0.0
    t_layer = ((((t_qkv + t_attp) + t_attd) + t_o) + t_up) + t_down     # step 2
    T = t_layer * float(L)                                              # step 3
    T = T + t_lm                                                        # step 4
    t = hw.tp_degree
    if t > 1:                                                           # step 5 (AR row, t > 1)
        invT = 1.0 / (float(t) * hw.tp_link_bw)
        b_ar = 2 * (t - 1) * N * h * s
        T = T + (float(b_ar) * invT) * float(2 * L)
    if swap_bytes > 0:                                                  # step 6 (+0.0 is exact)
        T = T + float(swap_bytes) * invH
    T = T + hw.iter_overhead_s                                          # step 7
    return int(math.floor(T * 1e9 + 0.5))                              # step 8


# ----------------------------------------------------------------------------- c.4 loop
@dataclass
class _Req:
    a: int
    p: int
    o: int
    ctx: int = 0
    gen: int = 0
    blocks: List[int] = field(default_factory=list)
    first: int = 0
    last: int = 0
    maxgap: int = 0
    npre: int = 0
    status: int = 0          # 0 unfinished, 1 finished, 2 rejected
    finish: int = 0
    finish_k: int = 0


def simulate(model, hw, pol, reqs: List[Tuple[int, int, int]], max_iters: int = 100000):
    """Run one point.  Returns dict(iters=[tuple], events=[(k, kind, req, block)],
    records=[(ttft, e2e, mtpot, n_preempt, status, finish_k)],
    victims=[(victim ids, (free count, [(id, need, held) of R])) per iteration],
    swap_out, swap_in)."""
    bs = pol.block_size
    total = hw.kv_blocks_override
    assert total > 0, "tiny reference: capacity via kv_blocks_override"
    ratio = pol.kind == "cont_ratio"
    static = pol.kind == "static"
    swap = pol.preempt == "swap"
    ratio_limit = int(math.floor(pol.max_mem_ratio * float(total)))
    kvb = 2 * model.num_layers * model.num_kv_heads * model.head_dim * model.dtype_bytes
    bb = bs * kvb
    mns, mbt, wm = pol.max_num_seqs, pol.max_batched_tokens, pol.watermark_blocks

    rq = [_Req(a, p, o) for (a, p, o) in reqs]
    n = len(rq)
    free = list(range(total))          # kept sorted: lowest index first
    R: List[int] = []                  # running, ascending id
    Q: List[int] = []                  # preempted, ascending id
    t = 0
    k = 0
    arr = adm = 0
    iters, events, victims_log = [], [], []
    swap_out_total = swap_in_total = 0

    def take(i: int, cnt: int):
        for _ in range(cnt):
            b = free.pop(0)
            rq[i].blocks.append(b)
            events.append((k, 1, i, b))

    def release(i: int):
        for b in rq[i].blocks:         # logical order
            free.append(b)
            events.append((k, 2, i, b))
        free.sort()
        rq[i].blocks = []

    while True:
        if adm == n and not R and not Q:                       # 0. termination
            break
        assert k < max_iters
        while arr < n and rq[arr].a <= t:                      # 1. ingest
            arr += 1
        if not R and not Q and adm == arr:                     # 2. idle skip
            t = rq[arr].a
            continue
        entry = {}                                             # id -> "dec" | "fresh" | "recomp"
        # 3. decode reservation, SEQUENTIAL rule on counts (vLLM: pop the latest while r can't fit)
        running = list(R)
        avail = len(free)
        pre = (avail, [(r, 1 if rq[r].ctx % bs == 0 else 0, len(rq[r].blocks)) for r in R])
        victims: List[int] = []
        j = 0
        while j < len(running):
            r = running[j]
            if rq[r].ctx % bs == 0:
                while avail == 0:
                    v = running.pop()                          # latest arrival still running
                    victims.append(v)
                    avail += len(rq[v].blocks)
                    if v == r:
                        break
                if r in victims:
                    break
                avail -= 1
            j += 1
        m = len(victims)
        swap_out = swap_in = 0
        for v in victims:                                      # A14: victim frees first
            x = rq[v]
            held = len(x.blocks)
            release(v)
            x.npre += 1
            if swap:
                swap_out += held * bb
            else:
                x.ctx = 0
            R.remove(v)
            Q.append(v)
        Q.sort()
        for r in R:                                            # then one block per needing survivor
            entry[r] = "dec"
            if rq[r].ctx % bs == 0:
                take(r, 1)
        tokens = len(R)
        n_res = n_adm = n_rej = 0
        if m == 0:
            for x_id in list(Q):                               # 4. resume, head first
                x = rq[x_id]
                if swap:
                    need = -(-x.ctx // bs) + (1 if x.ctx % bs == 0 else 0)
                    tok = 1
                else:
                    need = -(-(x.p + x.gen) // bs)
                    tok = x.p + x.gen
                if not (len(R) + 1 <= mns and tokens + tok <= mbt and len(free) - need >= wm):
                    break
                take(x_id, need)
                Q.remove(x_id)
                R.append(x_id)
                R.sort()
                n_res += 1
                tokens += tok
                if swap:
                    swap_in += -(-x.ctx // bs) * bb
                    entry[x_id] = "dec"
                else:
                    entry[x_id] = "recomp"
            if not Q and (not static or not R):                # 5. fresh FCFS admission
                while adm < arr:
                    x = rq[adm]
                    need = -(-x.p // bs)
                    cap = ratio_limit if ratio else total - wm
                    if need > cap:
                        x.status = 2
                        n_rej += 1
                        adm += 1
                        continue
                    if len(R) + 1 > mns or tokens + x.p > mbt or len(free) - need < wm:
                        break
                    if ratio and (total - len(free)) + need > ratio_limit:
                        break
                    take(adm, need)
                    R.append(adm)
                    R.sort()
                    entry[adm] = "fresh"
                    tokens += x.p
                    n_adm += 1
                    adm += 1
        if not entry:                                          # 6. empty batch
            continue
        ids = sorted(entry)
        pf, dec = [], []
        for i in ids:                                          # 7. cost
            x = rq[i]
            if entry[i] == "dec":
                dec.append(x.ctx + 1)
            elif entry[i] == "fresh":
                pf.append((x.p, 0))
            else:
                pf.append((x.p + x.gen, 0))
        T = cost_ns(model, hw, pf, dec, swap_out + swap_in)
        ts, te = t, t + T                                      # 8. commit
        blocks = total - len(free)
        n_fin = 0
        for i in ids:
            x = rq[i]
            if entry[i] == "fresh":
                x.ctx, x.gen, x.first, x.last = x.p, 1, te, te
            else:
                if entry[i] == "recomp":
                    x.ctx = x.p + x.gen
                else:
                    x.ctx += 1
                x.gen += 1
                x.maxgap = max(x.maxgap, te - x.last)
                x.last = te
            if x.gen == x.o:
                x.status, x.finish, x.finish_k = 1, te, k
                release(i)
                R.remove(i)
                n_fin += 1
        Np = sum(e[0] for e in pf)
        iters.append((k, ts, T, len(pf), len(dec), Np, sum(dec), m, n_res, n_adm, n_rej, n_fin, blocks))
        victims_log.append((victims, pre))
        swap_out_total += swap_out
        swap_in_total += swap_in
        t = te
        k += 1
    records = []
    for x in rq:
        fin = x.status == 1
        records.append((x.first - x.a if (x.gen >= 1 or fin) else 0, x.finish - x.a if fin else 0,
                        x.maxgap if fin else 0, x.npre, x.status, x.finish_k if fin else 0))
    return {"iters": iters, "events": events, "records": records, "victims": victims_log,
            "swap_out": swap_out_total, "swap_in": swap_in_total}
