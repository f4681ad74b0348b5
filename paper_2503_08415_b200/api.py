"""Python API of the B200 sweep -- thin marshalling over the C ABI (include/tokensim.h).

    from paper_2503_08415_b200 import Sweep
    import sweep_inputs as si
    sw = Sweep(si.c2())
    sw.run()                         # all points on the current CUDA device / stream
    s = sw.summaries()               # numpy structured array, one 384-B record per point

PyTorch provides device memory (the run workspace is a torch uint8 tensor), the
stream (torch.cuda.current_stream()) and, in ``run_distributed``, the process
group.  Every step of the sweep runs in the library's CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

import sweep_inputs as si

from . import _lib as T


class TokensimError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{T.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_KIND = {si.STATIC: T.STATIC, si.CONT: T.CONT, si.CONT_RATIO: T.CONT_RATIO}
_PRE = {si.SWAP: T.SWAP, si.RECOMPUTE: T.RECOMPUTE}
_DISPATCH = {si.ROUND_ROBIN: T.DISPATCH_ROUND_ROBIN, si.LEAST_OUTSTANDING: T.DISPATCH_LEAST_OUTSTANDING,
             si.LEAST_MEMORY: T.DISPATCH_LEAST_MEMORY}
_MODE = {si.MIXED: T.MIXED, si.PREFILL_FIRST: T.PREFILL_FIRST, si.CHUNKED: T.CHUNKED}
_LEN = {si.FIXED: T.LEN_FIXED, si.UNIFORM: T.LEN_UNIFORM, si.TABLE: T.LEN_TABLE, si.TRACE: T.LEN_TRACE,
        "sharegpt_synth_v1": T.LEN_SHAREGPT_SYNTH_V1}
_TRC = {si.NONE_TRACE: T.TRACE_NONE, si.BINNED: T.TRACE_BINNED, si.FULL: T.TRACE_FULL}
_TOP = {si.UNIFIED: T.UNIFIED, si.PD_PAIR: T.PD_PAIR}
METRICS = {"ttft": T.TTFT, "tpot": T.TPOT, "e2e": T.E2E, "norm": T.NORM, "mtpot": T.MTPOT}


def _arr(values, dtype, ctype):
    a = np.ascontiguousarray(np.asarray(values, dtype=dtype))
    return a, a.ctypes.data_as(C.POINTER(ctype))


def marshal(cfg: si.SweepConfig):
    """SweepConfig -> ctypes structs (+ keepalive list)."""
    keep = []
    m = cfg.model
    cm = T.Model(C.sizeof(T.Model), m.num_layers, m.hidden, m.num_heads, m.num_kv_heads, m.head_dim,
                 m.ffn_dim, m.vocab, m.dtype_bytes, m.gated_mlp, m.tied_embeddings, m.max_model_len)
    hws = (T.Hw * len(cfg.hws))()
    for i, h in enumerate(cfg.hws):
        hws[i] = T.Hw(C.sizeof(T.Hw), h.peak_flops, h.mem_bw, h.eff_flops, h.eff_bw, h.mem_capacity,
                      h.reserve_frac, h.iter_overhead_s, h.host_link_bw, h.tp_degree, h.tp_link_bw,
                      h.kv_blocks_override)
    pols = (T.Policy * len(cfg.policies))()
    for i, p in enumerate(cfg.policies):
        pols[i] = T.Policy(C.sizeof(T.Policy), _KIND[p.kind], _PRE[p.preempt], p.max_mem_ratio,
                           p.max_num_seqs, p.max_batched_tokens, p.block_size, p.watermark_blocks,
                           _MODE[p.iteration_mode])
    w = cfg.workload
    rates, prates = _arr(w.rates, np.float64, C.c_double)
    seeds, pseeds = _arr(w.seeds, np.uint64, C.c_uint64)
    keep += [rates, seeds, hws, pols]
    cw = T.Workload()
    cw.struct_size = C.sizeof(T.Workload)
    cw.num_requests = w.num_requests
    cw.num_rates, cw.rates = len(w.rates), prates
    cw.num_seeds, cw.seeds = len(w.seeds), pseeds
    cw.len_dist = _LEN[w.len_dist]
    cw.prompt_a, cw.prompt_b, cw.output_a, cw.output_b = w.prompt_a, w.prompt_b, w.output_a, w.output_b
    cw.multi_round, cw.think_mean_s = int(w.multi_round), w.think_mean_s
    if w.len_dist == si.TABLE:
        tabs = []
        for t in (w.prompt_table, w.output_table):
            lo, plo = _arr(t.lo, np.uint32, C.c_uint32)
            hi, phi = _arr(t.hi, np.uint32, C.c_uint32)
            th, pth = _arr(list(t.thr) + [0], np.uint32, C.c_uint32)
            lt = T.LenTable(len(t.lo), plo, phi, pth)
            keep += [lo, hi, th, lt]
            tabs.append(lt)
        cw.prompt_table = C.pointer(tabs[0])
        cw.output_table = C.pointer(tabs[1])
    if w.len_dist == si.TRACE:
        ta, pta = _arr(w.trace_arrival_ns, np.int64, C.c_int64)
        tp, ptp = _arr(w.trace_prompt, np.uint32, C.c_uint32)
        to, pto = _arr(w.trace_output, np.uint32, C.c_uint32)
        keep += [ta, tp, to]
        cw.trace_arrival_ns, cw.trace_prompt, cw.trace_output = pta, ptp, pto
    o = cfg.options
    flags = (0 if o.fast_forward else T.OPT_NO_FAST_FORWARD) | (T.OPT_NODE_LOOP if o.node_loop else 0)
    co = T.Options(C.sizeof(T.Options), _TOP[o.topology], o.pd_link_bw, _TRC[o.trace_mode], o.trace_bin_ns,
                   o.trace_cap_bytes, o.iteration_trace_cap, o.slo_ttft_s, o.slo_mtpot_s, o.horizon_ns,
                   flags, o.pd_prefill, o.pd_decode, _DISPATCH[o.dispatch],
                   {si.SEQUENTIAL: T.LINK_SEQUENTIAL, si.PRELOAD: T.LINK_PRELOAD}[o.link_mode], o.preload_buffer_bytes,
                   int(o.memory_cache), o.cache_capacity_blocks, o.cache_fetch_ns_per_block)
    return cm, hws, pols, cw, co, keep


class Sweep:
    """One sweep handle (tokensim_sweep)."""

    def __init__(self, cfg: si.SweepConfig):
        self.cfg = cfg
        self._L = T.lib()
        cm, hws, pols, cw, co, keep = marshal(cfg)
        h = C.c_void_p()
        st = self._L.tokensim_sweep_create(C.byref(cm), hws, len(cfg.hws), pols, len(cfg.policies),
                                           C.byref(cw), C.byref(co), C.byref(h))
        if st != T.OK:
            raise TokensimError(st, self._L.tokensim_last_error(None).decode())
        self._h = h
        self._ws = None
        self._n_req = cfg.workload.num_requests

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None):
            self._L.tokensim_sweep_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int, what: str):
        if st != T.OK:
            raise TokensimError(st, f"{what}: {self._L.tokensim_last_error(self._h).decode()}")

    @property
    def num_points(self) -> int:
        return int(self._L.tokensim_sweep_num_points(self._h))

    def workspace_size(self, begin: int = 0, end: Optional[int] = None, stride: int = 1) -> int:
        end = self.num_points if end is None else end
        b = C.c_size_t()
        self._check(self._L.tokensim_sweep_workspace_size(self._h, begin, end, stride, C.byref(b)), "workspace_size")
        return b.value

    def run(self, begin: int = 0, end: Optional[int] = None, stride: int = 1, device=None, stream=None,
            workspace=None):
        """Enqueue the sweep of points begin, begin+stride, ... < end on a CUDA stream.

        The workspace is a torch uint8 CUDA tensor (allocated here if not given) and
        stays referenced by this object until the next run."""
        import torch
        end = self.num_points if end is None else end
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        need = self.workspace_size(begin, end, stride)
        if workspace is None:
            if self._ws is None or self._ws.numel() < need or self._ws.device != dev:
                self._ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
            workspace = self._ws
        else:
            self._ws = workspace
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        st = self._L.tokensim_sweep_run(self._h, dev.index, begin, end, stride, C.c_void_p(workspace.data_ptr()),
                                        workspace.numel(), C.c_void_p(sptr))
        self._check(st, "run")
        return self

    # ------------------------------------------------------------------ results
    @property
    def num_run(self) -> int:
        return int(self._L.tokensim_sweep_num_run(self._h))

    def summaries(self) -> np.ndarray:
        n = C.c_uint64()
        self._check(self._L.tokensim_get_summaries(self._h, None, 0, C.byref(n)), "get_summaries")
        out = np.zeros(n.value, T.SUMMARY_DTYPE)
        if n.value:
            self._check(self._L.tokensim_get_summaries(self._h, out.ctypes.data, n.value, C.byref(n)),
                        "get_summaries")
        return out

    def summary(self, point: int) -> np.void:
        out = np.zeros(1, T.SUMMARY_DTYPE)
        self._check(self._L.tokensim_get_summary(self._h, point, out.ctypes.data), "get_summary")
        return out[0]

    def summaries_device(self):
        """torch uint8 view of the last run's summaries in device memory (for all-gather)."""
        p = C.c_void_p()
        b = C.c_size_t()
        self._check(self._L.tokensim_get_summaries_device(self._h, C.byref(p), C.byref(b)), "get_summaries_device")
        off = p.value - self._ws.data_ptr()
        return self._ws[off:off + b.value]

    def import_summaries(self, arr: np.ndarray):
        arr = np.ascontiguousarray(arr, dtype=T.SUMMARY_DTYPE)
        self._check(self._L.tokensim_import_summaries(self._h, arr.ctypes.data, arr.nbytes), "import_summaries")

    def records(self, point: int) -> np.ndarray:
        """Per-request records of one point (multi-round: one per round, rid order)."""
        n = C.c_uint64()
        self._check(self._L.tokensim_get_request_records(self._h, point, None, 0, C.byref(n)), "get_request_records")
        out = np.zeros(n.value, T.RECORD_DTYPE)
        self._check(self._L.tokensim_get_request_records(self._h, point, out.ctypes.data, len(out), C.byref(n)),
                    "get_request_records")
        return out

    def mem_trace(self, point: int, worker: int = 0, allow_overflow: bool = True) -> np.ndarray:
        n = C.c_uint64()
        self._check(self._L.tokensim_get_mem_trace(self._h, point, worker, None, 0, C.byref(n)), "get_mem_trace")
        out = np.zeros(n.value, T.SAMPLE_DTYPE)
        if n.value:
            st = self._L.tokensim_get_mem_trace(self._h, point, worker, out.ctypes.data, n.value, C.byref(n))
            if not (st == T.OK or (allow_overflow and st == T.E_OVERFLOW)):
                self._check(st, "get_mem_trace")
        return out

    def mem_trace_encoded(self, point: int, worker: int = 0):
        """The FULL trace's compressed byte stream as stored on the device (see tokensim.h):
        (uint8 array, number of iterations it encodes)."""
        nb, ns = C.c_uint64(), C.c_uint64()
        self._check(self._L.tokensim_get_mem_trace_encoded(self._h, point, worker, None, 0, C.byref(nb), C.byref(ns)),
                    "get_mem_trace_encoded")
        out = np.zeros(nb.value, np.uint8)
        if nb.value:
            st = self._L.tokensim_get_mem_trace_encoded(self._h, point, worker, out.ctypes.data, nb.value,
                                                        C.byref(nb), C.byref(ns))
            if st not in (T.OK, T.E_OVERFLOW):
                self._check(st, "get_mem_trace_encoded")
        return out, ns.value

    def iteration_trace(self, point: int) -> np.ndarray:
        n = C.c_uint64()
        self._check(self._L.tokensim_get_iteration_trace(self._h, point, None, 0, C.byref(n)), "get_iteration_trace")
        out = np.zeros(n.value, T.ITER_DTYPE)
        if n.value:
            self._check(self._L.tokensim_get_iteration_trace(self._h, point, out.ctypes.data, n.value, C.byref(n)),
                        "get_iteration_trace")
        return out

    def latency_quantiles(self, point: int, metric, q_bp: Sequence[int]) -> np.ndarray:
        metric = METRICS[metric] if isinstance(metric, str) else int(metric)
        q, pq = _arr(q_bp, np.uint32, C.c_uint32)
        out = np.zeros(len(q), np.float64)
        self._check(self._L.tokensim_get_latency_quantiles(self._h, point, metric, pq, len(q),
                                                           out.ctypes.data_as(C.POINTER(C.c_double))),
                    "get_latency_quantiles")
        return out

    def run_info(self) -> dict:
        ri = T.RunInfo()
        self._check(self._L.tokensim_get_run_info(self._h, C.byref(ri)), "get_run_info")
        return {n: getattr(ri, n) for n, _ in T.RunInfo._fields_}

    def point_profile(self, point: int) -> dict:
        pp = T.PointProfile()
        self._check(self._L.tokensim_get_point_profile(self._h, point, C.byref(pp)), "get_point_profile")
        d = {n: getattr(pp, n) for n, _ in T.PointProfile._fields_}
        d["stretch_phase_cycles"] = list(d["stretch_phase_cycles"])
        d["normal_phase_cycles"] = list(d["normal_phase_cycles"])
        d["ff_failed"] = list(d["ff_failed"])
        d["ff_cut"] = list(d["ff_cut"])
        return d

    def workload(self, point: int):
        """The point's generated requests (multi-round: 7 x conversations slots in rid order,
        arrival = round 0's time or round r's think gap; unused slots are zero)."""
        n = self._n_req * (7 if self.cfg.workload.multi_round else 1)
        a = np.zeros(n, np.int64)
        p = np.zeros(n, np.uint32)
        o = np.zeros(n, np.uint32)
        self._check(self._L.tokensim_get_workload(self._h, point, a.ctypes.data_as(C.POINTER(C.c_int64)),
                                                  p.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                  o.ctypes.data_as(C.POINTER(C.c_uint32)), n), "get_workload")
        return a, p, o


def version() -> str:
    return T.lib().tokensim_version().decode()


def sweep(cfg: si.SweepConfig, device=None) -> np.ndarray:
    """End-to-end convenience: create, run every point on one GPU, return host summaries."""
    sw = Sweep(cfg)
    try:
        sw.run(device=device)
        return sw.summaries()
    finally:
        sw.close()


def config_fingerprint(cfg: si.SweepConfig) -> str:
    """A stable hash of a sweep configuration (checkpoints refuse to resume another config)."""
    import hashlib
    return hashlib.sha256(repr(cfg).encode()).hexdigest()[:32]


def sweep_resumable(cfg: si.SweepConfig, path: str, chunk_points: int = 1024, device=None,
                    max_chunks: Optional[int] = None) -> np.ndarray:
    """Point-granular checkpoint / resume: run the sweep in chunks of
    `chunk_points` consecutive points, writing every finished chunk's summaries to the
    checkpoint `path` (.npz, replaced atomically); a rerun skips the chunks already there.
    `max_chunks` stops after that many new chunks (an interrupted job, for tests).  Returns the
    summaries of every finished point (all points once complete; unfinished rows are zero,
    with version 0)."""
    import os
    fp = config_fingerprint(cfg)
    npts = cfg.num_points
    nch = -(-npts // chunk_points)
    summ = np.zeros(npts, T.SUMMARY_DTYPE)
    done = np.zeros(nch, np.bool_)
    if os.path.exists(path):  # validated before any device work
        z = np.load(path, allow_pickle=False)
        if str(z["fingerprint"]) != fp or int(z["chunk_points"]) != chunk_points:
            raise ValueError(f"checkpoint {path} belongs to another sweep (config or chunking differs)")
        summ = np.ascontiguousarray(z["summaries"]).view(T.SUMMARY_DTYPE).reshape(npts).copy()
        done = z["done"].astype(np.bool_)
    sw = Sweep(cfg)
    try:
        ran = 0
        for c in range(nch):
            if done[c]:
                continue
            if max_chunks is not None and ran >= max_chunks:
                break
            b, e = c * chunk_points, min(npts, (c + 1) * chunk_points)
            sw.run(b, e, 1, device=device)
            summ[b:e] = sw.summaries()
            done[c] = True
            ran += 1
            tmp = path + ".tmp.npz"
            np.savez(tmp, fingerprint=np.array(fp), chunk_points=np.array(chunk_points),
                     summaries=summ.view(np.uint8), done=done)
            os.replace(tmp, path)
        return summ
    finally:
        sw.close()


def shard_range(num_points: int, rank: int, world: int):
    """Points owned by `rank`: p = rank (mod world)."""
    return rank, num_points, world


def gather_summaries(local, num_points: int, group=None):
    """All-gather every rank's 384-B point summaries (the sweep's only collective).

    `local` is a torch uint8 tensor (device summaries from `Sweep.summaries_device()`, NCCL)
    or a numpy SUMMARY_DTYPE array (host, e.g. gloo).  Each rank contributes a fixed-size
    slot of ceil(P / world) records (zero padding has version 0 and is dropped).
    Returns all summaries sorted by point."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    per = -(-num_points // world) * T.SUMMARY_DTYPE.itemsize
    if isinstance(local, np.ndarray):
        local = torch.from_numpy(np.ascontiguousarray(local).view(np.uint8).copy())
    buf = torch.zeros(per, dtype=torch.uint8, device=local.device)
    buf[:local.numel()] = local
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * per, dtype=torch.uint8, device=local.device)
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        out = torch.cat(parts)
    allv = out.cpu().numpy().view(T.SUMMARY_DTYPE)
    allv = allv[allv["version"] != 0]
    return np.sort(allv, order="point")


def run_distributed(cfg: si.SweepConfig, group=None):
    """One process per GPU: rank r runs points r, r+W, ...; the summaries of all points are
    then all-gathered (NCCL over NVLink) and imported so every rank can answer summary and
    P50/P90/P99/max queries for every point.  Returns (sweep handle, all summaries)."""
    import torch.distributed as dist
    import torch
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    sw = Sweep(cfg)
    b, e, s = shard_range(sw.num_points, rank, world)
    if b < e:
        sw.run(b, e, s)
        local = sw.summaries_device()
    else:  # more ranks than points: this rank owns none and joins the all-gather with padding only
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        local = torch.zeros(0, dtype=torch.uint8, device=dev)
    allv = gather_summaries(local, sw.num_points, group)
    sw.import_summaries(allv)
    return sw, allv
