"""ctypes mirror of include/tokensim.h -- argument marshalling only.

Loads the in-tree ``libtokensim.so`` (built by ``paper_2503_08415_b200.build``).
There is no fallback: if the library is missing, importing fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TOKENSIM_LIB") or os.path.join(_HERE, "libtokensim.so")  # env: A/B builds

u8, u16, u32, u64, i64, f64 = C.c_uint8, C.c_uint16, C.c_uint32, C.c_uint64, C.c_int64, C.c_double
PU32, PU64, PI64, PF64 = C.POINTER(u32), C.POINTER(u64), C.POINTER(i64), C.POINTER(f64)

# ---- enums (tokensim.h)
OK, E_INVALID, E_NOMEM, E_CUDA, E_STATE, E_RANGE, E_TRUNCATED, E_OVERFLOW = 0, -1, -2, -3, -4, -5, -6, -7
STATUS_NAMES = {0: "OK", -1: "E_INVALID", -2: "E_NOMEM", -3: "E_CUDA", -4: "E_STATE", -5: "E_RANGE",
                -6: "E_TRUNCATED", -7: "E_OVERFLOW"}
STATIC, CONT, CONT_RATIO = 0, 1, 2
SWAP, RECOMPUTE = 0, 1
MIXED, PREFILL_FIRST, CHUNKED = 0, 1, 2
LEN_SHAREGPT_SYNTH_V1, LEN_FIXED, LEN_UNIFORM, LEN_TABLE, LEN_TRACE = 0, 1, 2, 3, 4
TRACE_NONE, TRACE_BINNED, TRACE_FULL = 0, 1, 2
UNIFIED, PD_PAIR = 0, 1
TTFT, TPOT, E2E, NORM, MTPOT = 0, 1, 2, 3, 4
REQ_UNFINISHED, REQ_FINISHED, REQ_REJECTED = 0, 1, 2
OPT_NO_FAST_FORWARD, OPT_NODE_LOOP = 1, 2
DISPATCH_ROUND_ROBIN, DISPATCH_LEAST_OUTSTANDING, DISPATCH_LEAST_MEMORY = 0, 1, 2
LINK_SEQUENTIAL, LINK_PRELOAD = 0, 1
PT_TRACE_OVERFLOW, PT_ALL_REJECTED, PT_HORIZON_HIT, PT_INTERNAL_ERROR = 1, 2, 4, 16


class Model(C.Structure):
    _fields_ = [(n, u32) for n in ("struct_size", "num_layers", "hidden", "num_heads", "num_kv_heads",
                                   "head_dim", "ffn_dim", "vocab", "dtype_bytes", "gated_mlp",
                                   "tied_embeddings", "max_model_len")]


class Hw(C.Structure):
    _fields_ = [("struct_size", u32), ("peak_flops", f64), ("mem_bw", f64), ("eff_flops", f64),
                ("eff_bw", f64), ("mem_capacity", u64), ("reserve_frac", f64), ("iter_overhead_s", f64),
                ("host_link_bw", f64), ("tp_degree", u32), ("tp_link_bw", f64), ("kv_blocks_override", u64)]


class Policy(C.Structure):
    _fields_ = [("struct_size", u32), ("kind", u32), ("preempt", u32), ("max_mem_ratio", f64),
                ("max_num_seqs", u32), ("max_batched_tokens", u32), ("block_size", u32),
                ("watermark_blocks", u32), ("iteration_mode", u32)]


class LenTable(C.Structure):
    _fields_ = [("n_buckets", u32), ("lo", PU32), ("hi", PU32), ("cdf32", PU32)]


class Workload(C.Structure):
    _fields_ = [("struct_size", u32), ("num_requests", u32), ("num_rates", u32), ("rates", PF64),
                ("num_seeds", u32), ("seeds", PU64), ("len_dist", u32), ("prompt_a", u32),
                ("prompt_b", u32), ("output_a", u32), ("output_b", u32),
                ("prompt_table", C.POINTER(LenTable)), ("output_table", C.POINTER(LenTable)),
                ("trace_arrival_ns", PI64), ("trace_prompt", PU32), ("trace_output", PU32),
                ("multi_round", u32), ("think_mean_s", f64)]


class Options(C.Structure):
    _fields_ = [("struct_size", u32), ("topology", u32), ("pd_link_bw", f64), ("trace_mode", u32),
                ("trace_bin_ns", u64), ("trace_cap_bytes", u64), ("iteration_trace_cap", u32),
                ("slo_ttft_s", f64), ("slo_mtpot_s", f64), ("horizon_ns", i64), ("flags", u32),
                ("pd_prefill_workers", u32), ("pd_decode_workers", u32), ("dispatch", u32),
                ("link_mode", u32), ("preload_buffer_bytes", u64),
                ("memory_cache", u32), ("cache_capacity_blocks", u64), ("cache_fetch_ns_per_block", f64)]


class PointProfile(C.Structure):
    _fields_ = [("n_iterations", u64), ("ff_iterations", u64), ("ff_stretches", u64), ("sm_cycles", u64),
                ("cycles_ff", u64), ("cycles_ff_failed", u64), ("cycles_normal", u64),
                ("stretch_phase_cycles", u64 * 8), ("n_transfers", u64), ("transfer_bytes", u64),
                ("normal_phase_cycles", u64 * 8), ("ff_failed", u64 * 5), ("ff_cut", u64 * 5)]


class RunInfo(C.Structure):
    _fields_ = [("ms_workload", f64), ("ms_sim", f64), ("ms_summary", f64), ("n_launches", u32),
                ("sim_blocks", u32), ("sim_warps_per_block", u32), ("smem_per_warp", u32), ("n_run", u64),
                ("h2d_bytes", u64), ("workspace_bytes", u64), ("helper_mode", u32), ("n_heads", u32)]


RECORD_DTYPE = np.dtype([("ttft_ns", "<i8"), ("e2e_ns", "<i8"), ("mtpot_ns", "<i8"), ("n_preempt", "<u2"),
                         ("status", "u1"), ("pad", "u1"), ("finish_iter", "<u4")])
SAMPLE_DTYPE = np.dtype([("t_ns", "<i8"), ("dur_ns", "<i8"), ("block_ns", "<u8"), ("blocks_max", "<u4"),
                         ("n_iter", "<u4")])
ITER_DTYPE = np.dtype([("k", "<u8"), ("t_start_ns", "<i8"), ("T_ns", "<i8"), ("n_prefill", "<u4"),
                       ("n_decode", "<u4"), ("N_p", "<u8"), ("C_d", "<u8"), ("n_preempted", "<u4"),
                       ("n_resumed", "<u4"), ("n_admitted", "<u4"), ("n_rejected", "<u4"),
                       ("n_finished", "<u4"), ("blocks_in_use", "<u4"), ("worker", "<u4"), ("pad", "<u4")])
SUMMARY_DTYPE = np.dtype([
    ("version", "<u4"), ("status_flags", "<u4"), ("point", "<u8"),
    ("n_requests", "<u8"), ("n_finished", "<u8"), ("n_rejected", "<u8"), ("n_unfinished", "<u8"),
    ("n_iterations", "<u8"), ("n_request_iterations", "<u8"), ("n_preemptions", "<u8"),
    ("swap_out_bytes", "<u8"), ("swap_in_bytes", "<u8"),
    ("first_arrival_ns", "<i8"), ("last_finish_ns", "<i8"),
    ("sched_digest", "<u8"), ("block_digest", "<u8"), ("request_digest", "<u8"),
    ("total_blocks", "<u4"), ("peak_blocks", "<u4"), ("mean_util", "<f8"),
    ("stat", "<f8", (5, 5)),
    ("throughput_rps", "<f8"), ("goodput_mtpot_rps", "<f8"), ("goodput_both_rps", "<f8"),
    ("t_final_ns", "<i8"), ("block_ns_sum", "<u8"),
])
assert RECORD_DTYPE.itemsize == 32 and SAMPLE_DTYPE.itemsize == 32
assert ITER_DTYPE.itemsize == 80 and SUMMARY_DTYPE.itemsize == 384

EXPORTS = [
    "tokensim_sweep_create", "tokensim_sweep_num_points", "tokensim_sweep_workspace_size", "tokensim_sweep_run",
    "tokensim_sweep_num_run", "tokensim_get_latency_quantiles", "tokensim_get_mem_trace", "tokensim_get_summary",
    "tokensim_get_summaries", "tokensim_get_summaries_device", "tokensim_import_summaries",
    "tokensim_get_request_records", "tokensim_get_iteration_trace", "tokensim_get_workload",
    "tokensim_last_error", "tokensim_sweep_destroy", "tokensim_version", "tokensim_get_run_info",
    "tokensim_get_point_profile", "tokensim_get_mem_trace_encoded",
]

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2503_08415_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.tokensim_sweep_create.argtypes = [C.POINTER(Model), C.POINTER(Hw), u32, C.POINTER(Policy), u32,
                                        C.POINTER(Workload), C.POINTER(Options), C.POINTER(vp)]
    L.tokensim_sweep_create.restype = C.c_int
    L.tokensim_sweep_num_points.argtypes = [vp]
    L.tokensim_sweep_num_points.restype = u64
    L.tokensim_sweep_num_run.argtypes = [vp]
    L.tokensim_sweep_num_run.restype = u64
    L.tokensim_sweep_workspace_size.argtypes = [vp, u64, u64, u64, C.POINTER(C.c_size_t)]
    L.tokensim_sweep_workspace_size.restype = C.c_int
    L.tokensim_sweep_run.argtypes = [vp, C.c_int, u64, u64, u64, vp, C.c_size_t, vp]
    L.tokensim_sweep_run.restype = C.c_int
    L.tokensim_get_latency_quantiles.argtypes = [vp, u64, u32, PU32, u32, PF64]
    L.tokensim_get_latency_quantiles.restype = C.c_int
    L.tokensim_get_mem_trace.argtypes = [vp, u64, u32, vp, u64, PU64]
    L.tokensim_get_mem_trace.restype = C.c_int
    L.tokensim_get_mem_trace_encoded.argtypes = [vp, u64, u32, vp, u64, PU64, PU64]
    L.tokensim_get_mem_trace_encoded.restype = C.c_int
    L.tokensim_get_summary.argtypes = [vp, u64, vp]
    L.tokensim_get_summary.restype = C.c_int
    L.tokensim_get_summaries.argtypes = [vp, vp, u64, PU64]
    L.tokensim_get_summaries.restype = C.c_int
    L.tokensim_get_summaries_device.argtypes = [vp, C.POINTER(vp), C.POINTER(C.c_size_t)]
    L.tokensim_get_summaries_device.restype = C.c_int
    L.tokensim_import_summaries.argtypes = [vp, vp, C.c_size_t]
    L.tokensim_import_summaries.restype = C.c_int
    L.tokensim_get_request_records.argtypes = [vp, u64, vp, u64, PU64]
    L.tokensim_get_request_records.restype = C.c_int
    L.tokensim_get_iteration_trace.argtypes = [vp, u64, vp, u64, PU64]
    L.tokensim_get_iteration_trace.restype = C.c_int
    L.tokensim_get_workload.argtypes = [vp, u64, PI64, PU32, PU32, u64]
    L.tokensim_get_workload.restype = C.c_int
    L.tokensim_last_error.argtypes = [vp]
    L.tokensim_last_error.restype = C.c_char_p
    L.tokensim_sweep_destroy.argtypes = [vp]
    L.tokensim_sweep_destroy.restype = None
    L.tokensim_version.restype = C.c_char_p
    L.tokensim_get_run_info.argtypes = [vp, C.POINTER(RunInfo)]
    L.tokensim_get_run_info.restype = C.c_int
    L.tokensim_get_point_profile.argtypes = [vp, u64, C.POINTER(PointProfile)]
    L.tokensim_get_point_profile.restype = C.c_int
    _lib = L
    return L
