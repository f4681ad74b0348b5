"""Parity helpers: run the oracle on grid points (process pool) and compare its results
with the CUDA path element by element.  Test infrastructure only."""
from __future__ import annotations

import concurrent.futures as cf
import multiprocessing as mp
import os
from typing import Dict, Iterable, List

import numpy as np

import sweep_inputs as si

EXACT_FIELDS = ["n_requests", "n_finished", "n_rejected", "n_unfinished", "n_iterations", "n_request_iterations",
                "n_preemptions", "swap_out_bytes", "swap_in_bytes", "first_arrival_ns", "last_finish_ns",
                "sched_digest", "block_digest", "request_digest", "total_blocks", "peak_blocks", "block_ns_sum",
                "status_flags"]
FP_FIELDS = ["mean_util", "throughput_rps", "goodput_mtpot_rps", "goodput_both_rps"]
REL_TOL = 1e-9   # BASELINE.json north_star: fp64 latencies/quantiles within 1e-9 relative


def _oracle_job(args):
    cfg, point, want = args
    from oracle import oracle as O
    return point, O.simulate(cfg, point, want=want)


def oracle_points(cfg: si.SweepConfig, points: Iterable[int], want=("summary", "records"),
                  procs: int = 0) -> Dict[int, dict]:
    points = list(points)
    procs = procs or min(len(points), max(1, len(os.sched_getaffinity(0))))
    if procs <= 1 or len(points) <= 1:
        return dict(_oracle_job((cfg, p, want)) for p in points)
    ctx = mp.get_context("spawn")
    with cf.ProcessPoolExecutor(procs, mp_context=ctx) as ex:
        return dict(ex.map(_oracle_job, [(cfg, p, want) for p in points]))


TRACE_OVERFLOW = 1


def compare_summary(g, o: dict, point: int, full_trace: bool = False) -> List[str]:
    """full_trace: the CUDA path's FULL trace is a compressed stream with a byte budget, the
    oracle keeps every sample; the overflow bit is then the CUDA side's own (see compare_trace)."""
    bad = []
    for f in EXACT_FIELDS:
        gv, ov = int(g[f]), int(o[f])
        if f == "status_flags" and full_trace:
            gv, ov = gv & ~TRACE_OVERFLOW, ov & ~TRACE_OVERFLOW
        if gv != ov:
            bad.append(f"point {point}: {f} gpu={gv} oracle={ov}")
    if int(g["t_final_ns"]) != int(o["t_final"]):
        bad.append(f"point {point}: t_final gpu={int(g['t_final_ns'])} oracle={int(o['t_final'])}")
    for f in FP_FIELDS:
        if not _close(float(g[f]), float(o[f])):
            bad.append(f"point {point}: {f} gpu={float(g[f])!r} oracle={float(o[f])!r}")
    gs, os_ = np.asarray(g["stat"]), np.asarray(o["stat"])
    for m in range(5):
        for q in range(5):
            if not _close(float(gs[m, q]), float(os_[m, q])):
                bad.append(f"point {point}: stat[{m}][{q}] gpu={gs[m, q]!r} oracle={os_[m, q]!r}")
    return bad


def _close(a: float, b: float) -> bool:
    return a == b or abs(a - b) <= REL_TOL * max(abs(a), abs(b))


def compare_records(g: np.ndarray, o: np.ndarray, point: int) -> List[str]:
    bad = []
    if len(g) != len(o):
        return [f"point {point}: record count {len(g)} != {len(o)}"]
    for f, of in (("ttft_ns", "ttft_ns"), ("e2e_ns", "e2e_ns"), ("mtpot_ns", "mtpot_ns"),
                  ("n_preempt", "n_preempt"), ("status", "status")):
        gv = g[f].astype(np.int64)
        ov = o[of].astype(np.int64)
        d = np.nonzero(gv != ov)[0]
        if len(d):
            i = int(d[0])
            bad.append(f"point {point}: {len(d)} records differ in {f}; first id {i}: gpu={gv[i]} oracle={ov[i]}")
    fk = (o["finish_k"] & 0xFFFFFFFF).astype(np.int64)
    d = np.nonzero(g["finish_iter"].astype(np.int64) != fk)[0]
    if len(d):
        bad.append(f"point {point}: finish_iter differs for {len(d)} records (first {int(d[0])})")
    return bad


def compare_trace(g: np.ndarray, o: np.ndarray, point: int, prefix: bool = False) -> List[str]:
    """prefix: the CUDA FULL stream overflowed its byte budget; it must hold exactly the
    oracle's first len(g) samples."""
    if prefix and len(g) <= len(o):
        o = o[:len(g)]
    if len(g) != len(o):
        return [f"point {point}: trace length gpu={len(g)} oracle={len(o)}"]
    bad = []
    for f in ("t_ns", "dur_ns", "block_ns", "blocks_max", "n_iter"):
        d = np.nonzero(g[f].astype(np.int64) != o[f].astype(np.int64))[0]
        if len(d):
            bad.append(f"point {point}: trace {f} differs at {len(d)} samples (first {int(d[0])})")
    return bad


def compare_iters(g: np.ndarray, o: np.ndarray, point: int) -> List[str]:
    n = min(len(g), len(o))
    pairs = [("k", "k"), ("t_start_ns", "t_start"), ("T_ns", "T_ns"), ("n_prefill", "S_p"), ("n_decode", "D"),
             ("N_p", "N_p"), ("C_d", "C_d"), ("n_preempted", "m"), ("n_resumed", "n_resumed"),
             ("n_admitted", "n_admitted"), ("n_rejected", "n_rejected"), ("n_finished", "n_finished"),
             ("blocks_in_use", "blocks")]
    for i in range(n):
        for gf, of in pairs:
            if int(g[gf][i]) != int(o[of][i]):
                return [f"point {point}: first divergent iteration {i}: {gf} gpu={int(g[gf][i])} "
                        f"oracle={int(o[of][i])}"]
    if len(g) != len(o):
        return [f"point {point}: iteration count gpu={len(g)} oracle={len(o)}"]
    return []


def sample_points(num_points: int, target: int = 64, corners=()) -> List[int]:
    """Deterministic sample S = {p : p mod ceil(P/target) == 0} u corners."""
    step = max(1, -(-num_points // target))
    s = set(range(0, num_points, step)) | {c for c in corners if 0 <= c < num_points} | {num_points - 1}
    return sorted(s)
