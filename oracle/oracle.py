"""ctypes binding of liboracle.so -- the CPU oracle (TEST INFRASTRUCTURE ONLY).

Builds ``oracle/liboracle.so`` from ``oracle.cpp`` with
``g++ -std=c++17 -O2 -ffp-contract=off`` (no fast-math, no FMA contraction),
marshals a ``sweep_inputs.SweepConfig`` grid point into the oracle's own
``oracle_cfg`` struct, and returns plain numpy/dict results.  The point-grid
decode (SURVEY §8(b) "Point grid") is done here independently of the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, Optional

import numpy as np

import sweep_inputs as si

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

GXX_FLAGS = ["-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile liboracle.so if missing or older than its sources."""
    stale = force or not os.path.exists(_LIB) or max(
        os.path.getmtime(_SRC), os.path.getmtime(_HDR)) > os.path.getmtime(_LIB)
    if stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *GXX_FLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


u32, u64, i64, f64 = C.c_uint32, C.c_uint64, C.c_int64, C.c_double
PU32, PI64 = C.POINTER(u32), C.POINTER(i64)


class OracleCfg(C.Structure):
    _fields_ = [
        *[(n, u32) for n in ("L", "h", "n_heads", "n_kv", "head_dim", "ffn", "vocab",
                             "dtype_bytes", "gated", "tied", "max_model_len")],
        ("peak_flops", f64), ("mem_bw", f64), ("eff_flops", f64), ("eff_bw", f64),
        ("mem_capacity", u64), ("reserve_frac", f64), ("iter_overhead_s", f64),
        ("host_link_bw", f64), ("tp_degree", u32), ("tp_link_bw", f64),
        ("kv_blocks_override", u64),
        ("d_peak_flops", f64), ("d_mem_bw", f64), ("d_eff_flops", f64), ("d_eff_bw", f64),
        ("d_mem_capacity", u64), ("d_reserve_frac", f64), ("d_iter_overhead_s", f64),
        ("d_host_link_bw", f64), ("d_tp_degree", u32), ("d_tp_link_bw", f64),
        ("d_kv_blocks_override", u64),
        ("kind", u32), ("preempt", u32), ("max_mem_ratio", f64),
        ("max_num_seqs", u32), ("max_batched_tokens", u32), ("block_size", u32),
        ("watermark_blocks", u32),
        ("num_requests", u32), ("rate", f64), ("seed", u64),
        ("len_dist", u32), ("prompt_a", u32), ("prompt_b", u32), ("output_a", u32), ("output_b", u32),
        ("pt_n", u32), ("pt_lo", PU32), ("pt_hi", PU32), ("pt_thr", PU32),
        ("ot_n", u32), ("ot_lo", PU32), ("ot_hi", PU32), ("ot_thr", PU32),
        ("trace_arrival_ns", PI64), ("trace_prompt", PU32), ("trace_output", PU32),
        ("topology", u32), ("pd_link_bw", f64), ("trace_mode", u32),
        ("trace_bin_ns", u64), ("trace_cap_samples", u64),
        ("slo_ttft_s", f64), ("slo_mtpot_s", f64), ("horizon_ns", i64),
        ("check_invariants", u32), ("keep_events", u32), ("iter_mode", u32),
        ("n_prefill", u32), ("n_decode", u32), ("dispatch", u32), ("force_general", u32),
        ("link_mode", u32), ("preload_buffer_bytes", u64),
        ("multi_round", u32), ("think_mean_s", f64), ("memory_cache", u32), ("cache_capacity_blocks", u64),
        ("cache_fetch_ns_per_block", f64),
    ]


class OracleDerived(C.Structure):
    _fields_ = [(n, u64) for n in ("W", "kvb", "block_bytes", "reserve", "total_blocks", "ratio_limit")] + \
               [(n, f64) for n in ("invF", "invB", "invH", "invT", "scale_ns")] + \
               [("slo_ttft_ns", i64), ("slo_mtpot_ns", i64)]


RECORD_DTYPE = np.dtype([("ttft_ns", "<i8"), ("e2e_ns", "<i8"), ("mtpot_ns", "<i8"),
                         ("n_preempt", "<u4"), ("status", "<u4"), ("finish_k", "<u8")])
ITER_DTYPE = np.dtype([("k", "<u8"), ("t_start", "<i8"), ("T_ns", "<i8")] +
                      [(n, "<u8") for n in ("S_p", "D", "N_p", "C_d", "m", "n_resumed", "n_admitted",
                                            "n_rejected", "n_finished", "blocks")] +
                      [("worker", "<u4"), ("pad", "<u4")])
SAMPLE_DTYPE = np.dtype([("t_ns", "<i8"), ("dur_ns", "<i8"), ("block_ns", "<u8"),
                         ("blocks_max", "<u4"), ("n_iter", "<u4")])
EVENT_DTYPE = np.dtype([("k", "<u8"), ("kind", "<u4"), ("req", "<u4"), ("block", "<u4"), ("worker", "<u4")])


class OracleSummary(C.Structure):
    _fields_ = [("status_flags", u32)] + \
        [(n, u64) for n in ("n_requests", "n_finished", "n_rejected", "n_unfinished", "n_iterations",
                            "n_request_iterations", "n_preemptions", "swap_out_bytes", "swap_in_bytes")] + \
        [("first_arrival_ns", i64), ("last_finish_ns", i64), ("t_final", i64)] + \
        [(n, u64) for n in ("sched_digest", "block_digest", "request_digest", "total_blocks",
                            "peak_blocks", "block_ns_sum")] + \
        [("mean_util", f64), ("stat", (f64 * 5) * 5), ("throughput_rps", f64),
         ("goodput_mtpot_rps", f64), ("goodput_both_rps", f64),
         ("n_transfers", u64), ("transfer_bytes", u64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        L.oracle_philox4x32_10.argtypes = [PU32, PU32, PU32]
        L.oracle_det_log.argtypes = [f64]
        L.oracle_det_log.restype = f64
        L.oracle_derive.argtypes = [C.POINTER(OracleCfg), C.c_int, C.POINTER(OracleDerived)]
        L.oracle_derive.restype = C.c_int
        L.oracle_workload.argtypes = [C.POINTER(OracleCfg), PI64, PU32, PU32]
        L.oracle_workload.restype = C.c_int
        L.oracle_iter_time_ns.argtypes = [C.POINTER(OracleCfg), C.c_int, u32, PU32, PU32, PU32, u32, PU32, u64, u64]
        L.oracle_pipeline.argtypes = [u64, C.c_double, C.c_double, u64]
        L.oracle_workload_rounds.argtypes = [C.POINTER(OracleCfg), PI64, PU32, PU32, PU32]
        L.oracle_workload_rounds.restype = i64
        L.oracle_pipeline.restype = C.c_double
        L.oracle_iter_time_ns.restype = i64
        L.oracle_fold.argtypes = [C.POINTER(u64), u32]
        L.oracle_fold.restype = u64
        L.oracle_simulate.argtypes = [C.POINTER(OracleCfg)]
        L.oracle_simulate.restype = C.c_void_p
        L.oracle_error.restype = C.c_char_p
        L.oracle_summary_get.argtypes = [C.c_void_p, C.POINTER(OracleSummary)]
        for fn in ("oracle_records", "oracle_iters", "oracle_events"):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_void_p]
            getattr(L, fn).restype = u64
        L.oracle_trace.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.oracle_trace.restype = u64
        L.oracle_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


_KIND = {si.STATIC: 0, si.CONT: 1, si.CONT_RATIO: 2}
_PRE = {si.SWAP: 0, si.RECOMPUTE: 1}
_LEN = {si.FIXED: 1, si.UNIFORM: 2, si.TABLE: 3, si.TRACE: 4}
_TRC = {si.NONE_TRACE: 0, si.BINNED: 1, si.FULL: 2}


def _u32arr(v):
    a = np.ascontiguousarray(np.asarray(v, dtype=np.uint32))
    return a, a.ctypes.data_as(PU32)


def _set_hw(c: OracleCfg, hw: si.Hw, prefix: str = ""):
    for name in ("peak_flops", "mem_bw", "eff_flops", "eff_bw", "mem_capacity", "reserve_frac",
                 "iter_overhead_s", "host_link_bw", "tp_degree", "tp_link_bw", "kv_blocks_override"):
        setattr(c, prefix + name, getattr(hw, name))


def make_cfg(cfg: si.SweepConfig, point: int, check_invariants: bool = False,
             keep_events: bool = False, trace_cap_samples: Optional[int] = None):
    """Build the oracle struct for one grid point.  Returns (struct, keepalive)."""
    m, w, o = cfg.model, cfg.workload, cfg.options
    ns, nr, npol = len(w.seeds), len(w.rates), len(cfg.policies)
    seed_i = point % ns
    rate_i = (point // ns) % nr
    pol_i = (point // (ns * nr)) % npol
    hw_i = point // (ns * nr * npol)
    c = OracleCfg()
    keep = []
    c.L, c.h, c.n_heads, c.n_kv, c.head_dim = m.num_layers, m.hidden, m.num_heads, m.num_kv_heads, m.head_dim
    c.ffn, c.vocab, c.dtype_bytes, c.gated, c.tied = m.ffn_dim, m.vocab, m.dtype_bytes, m.gated_mlp, m.tied_embeddings
    c.max_model_len = m.max_model_len
    if o.topology == si.PD_PAIR:
        nh = len(cfg.hws)
        _set_hw(c, cfg.hws[hw_i // nh])
        _set_hw(c, cfg.hws[hw_i % nh], "d_")
        c.topology = 1
    else:
        _set_hw(c, cfg.hws[hw_i])
        _set_hw(c, cfg.hws[hw_i], "d_")
        c.topology = 0
    p = cfg.policies[pol_i]
    c.kind, c.preempt, c.max_mem_ratio = _KIND[p.kind], _PRE[p.preempt], p.max_mem_ratio
    c.max_num_seqs, c.max_batched_tokens = p.max_num_seqs, p.max_batched_tokens
    c.block_size, c.watermark_blocks = p.block_size, p.watermark_blocks
    c.iter_mode = {si.MIXED: 0, si.PREFILL_FIRST: 1, si.CHUNKED: 2}[p.iteration_mode]
    c.num_requests, c.rate, c.seed = w.num_requests, w.rates[rate_i], w.seeds[seed_i]
    c.len_dist = _LEN[w.len_dist]
    c.prompt_a, c.prompt_b, c.output_a, c.output_b = w.prompt_a, w.prompt_b, w.output_a, w.output_b
    if w.len_dist == si.TABLE:
        for pre, t in (("pt_", w.prompt_table), ("ot_", w.output_table)):
            a_lo, p_lo = _u32arr(t.lo)
            a_hi, p_hi = _u32arr(t.hi)
            a_th, p_th = _u32arr(list(t.thr) + [0])
            keep += [a_lo, a_hi, a_th]
            setattr(c, pre + "n", len(t.lo))
            setattr(c, pre + "lo", p_lo)
            setattr(c, pre + "hi", p_hi)
            setattr(c, pre + "thr", p_th)
    if w.len_dist == si.TRACE:
        ta = np.ascontiguousarray(np.asarray(w.trace_arrival_ns, dtype=np.int64))
        tp, pp = _u32arr(w.trace_prompt)
        to, po = _u32arr(w.trace_output)
        keep += [ta, tp, to]
        c.trace_arrival_ns = ta.ctypes.data_as(PI64)
        c.trace_prompt, c.trace_output = pp, po
    c.pd_link_bw = o.pd_link_bw
    c.trace_mode = _TRC[o.trace_mode]
    c.trace_bin_ns = o.trace_bin_ns
    # BINNED: the caller's cap in 32-B samples.  FULL: every iteration is kept (the CUDA path stores
    # FULL compressed, so its cap is a byte budget; parity compares the prefix it holds)
    if trace_cap_samples is None:
        trace_cap_samples = (1 << 40) if o.trace_mode == si.FULL else o.trace_cap_bytes // 32
    c.trace_cap_samples = trace_cap_samples
    c.slo_ttft_s, c.slo_mtpot_s, c.horizon_ns = o.slo_ttft_s, o.slo_mtpot_s, o.horizon_ns
    c.check_invariants = 1 if check_invariants else 0
    c.keep_events = 1 if keep_events else 0
    c.n_prefill, c.n_decode = o.pd_prefill, o.pd_decode
    c.link_mode = {si.SEQUENTIAL: 0, si.PRELOAD: 1}[o.link_mode]
    c.multi_round, c.think_mean_s = int(w.multi_round), w.think_mean_s
    c.memory_cache, c.cache_capacity_blocks = int(o.memory_cache), o.cache_capacity_blocks
    c.cache_fetch_ns_per_block = o.cache_fetch_ns_per_block
    c.preload_buffer_bytes = o.preload_buffer_bytes
    c.dispatch = {si.ROUND_ROBIN: 0, si.LEAST_OUTSTANDING: 1, si.LEAST_MEMORY: 2}[o.dispatch]
    return c, keep


def summary_to_dict(s: OracleSummary) -> Dict:
    d = {}
    for name, _ in OracleSummary._fields_:
        v = getattr(s, name)
        if name == "stat":
            v = np.array([[v[i][j] for j in range(5)] for i in range(5)])
        d[name] = v
    return d


def simulate(cfg: si.SweepConfig, point: int, check_invariants: bool = False,
             keep_events: bool = False, want=("summary", "records"), force_general: bool = False) -> Dict:
    """Run one grid point in the oracle; returns a dict of numpy arrays / summary."""
    L = lib()
    c, keep = make_cfg(cfg, point, check_invariants, keep_events)
    c.force_general = 1 if force_general else 0
    h = L.oracle_simulate(C.byref(c))
    if not h:
        raise OracleError(L.oracle_error().decode())
    try:
        out = {"point": point}
        s = OracleSummary()
        L.oracle_summary_get(h, C.byref(s))
        out["summary"] = summary_to_dict(s)
        if "records" in want:
            n = L.oracle_records(h, None)
            a = np.zeros(n, RECORD_DTYPE)
            L.oracle_records(h, a.ctypes.data)
            out["records"] = a
        if "iters" in want:
            n = L.oracle_iters(h, None)
            a = np.zeros(n, ITER_DTYPE)
            L.oracle_iters(h, a.ctypes.data)
            out["iters"] = a
        if "trace" in want:
            tr = []
            nw = cfg.options.pd_prefill + cfg.options.pd_decode if cfg.options.topology == si.PD_PAIR else 2
            for wk in range(nw):
                n = L.oracle_trace(h, wk, None)
                a = np.zeros(n, SAMPLE_DTYPE)
                L.oracle_trace(h, wk, a.ctypes.data)
                tr.append(a)
            out["trace"] = tr
        if "events" in want or keep_events:
            n = L.oracle_events(h, None)
            a = np.zeros(n, EVENT_DTYPE)
            L.oracle_events(h, a.ctypes.data)
            out["events"] = a
        return out
    finally:
        L.oracle_free(h)


def philox(ctr, key):
    L = lib()
    c = (u32 * 4)(*ctr)
    k = (u32 * 2)(*key)
    o = (u32 * 4)()
    L.oracle_philox4x32_10(c, k, o)
    return tuple(o)


def det_log(u: float) -> float:
    return lib().oracle_det_log(u)


def derive(cfg: si.SweepConfig, point: int = 0, decode_worker: int = 0) -> Dict:
    L = lib()
    c, keep = make_cfg(cfg, point)
    d = OracleDerived()
    if L.oracle_derive(C.byref(c), decode_worker, C.byref(d)) != 0:
        raise OracleError(L.oracle_error().decode())
    return {n: getattr(d, n) for n, _ in OracleDerived._fields_}


def workload(cfg: si.SweepConfig, point: int = 0):
    L = lib()
    c, keep = make_cfg(cfg, point)
    n = c.num_requests
    a = np.zeros(n, np.int64)
    p = np.zeros(n, np.uint32)
    o = np.zeros(n, np.uint32)
    if L.oracle_workload(C.byref(c), a.ctypes.data_as(PI64), p.ctypes.data_as(PU32),
                         o.ctypes.data_as(PU32)) != 0:
        raise OracleError(L.oracle_error().decode())
    return a, p, o


def workload_rounds(cfg: si.SweepConfig, point: int = 0):
    """NEXT-2 multi-round stream of one point: (arrival_or_think, prompt, output, conv) per request."""
    L = lib()
    c, keep = make_cfg(cfg, point)
    cap = 7 * c.num_requests
    a = np.zeros(cap, np.int64)
    p = np.zeros(cap, np.uint32)
    o = np.zeros(cap, np.uint32)
    cv = np.zeros(cap, np.uint32)
    n = L.oracle_workload_rounds(C.byref(c), a.ctypes.data_as(PI64), p.ctypes.data_as(PU32),
                                 o.ctypes.data_as(PU32), cv.ctypes.data_as(PU32))
    if n < 0:
        raise OracleError(L.oracle_error().decode())
    return a[:n], p[:n], o[:n], cv[:n]


def iter_time_ns(cfg: si.SweepConfig, prefills=(), decodes=(), swap_bytes: int = 0,
                 point: int = 0, decode_worker: int = 0, swap_in: int = 0) -> int:
    """T_ns of one explicit batch: prefills = [(P, c0) or (P, c0, emits), ...], decodes = [c, ...]."""
    L = lib()
    c, keep = make_cfg(cfg, point)
    P, pP = _u32arr([x[0] for x in prefills] or [0])
    c0, pc0 = _u32arr([x[1] for x in prefills] or [0])
    em, pem = _u32arr([int(x[2]) if len(x) > 2 else 1 for x in prefills] or [1])
    dc, pdc = _u32arr(list(decodes) or [0])
    return L.oracle_iter_time_ns(C.byref(c), decode_worker, len(prefills), pP, pc0, pem, len(decodes), pdc,
                                 swap_bytes, swap_in)


def pipeline(n_chunks: int, a: float, b: float, slots: int) -> float:
    """NEXT-4 preload pipeline completion time (see oracle.h)."""
    return lib().oracle_pipeline(n_chunks, a, b, slots)


def fold(fields) -> int:
    arr = (u64 * len(fields))(*[int(x) & 0xFFFFFFFFFFFFFFFF for x in fields])
    return lib().oracle_fold(arr, len(fields))
