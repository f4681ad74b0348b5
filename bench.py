#!/usr/bin/env python
"""Benchmark of the B200 batched design-space sweep (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One *step* = one pass of the whole hot path (workload
generation, the persistent per-point simulation kernel, the quantile/summary kernel)
over the configuration's sweep points.  The default workload is north_star's target, the
largest single-GPU configuration: BASELINE.json configs[2] = C3 (LLaMA-2-7B hardware sweep,
16 FLOP/s x 16 HBM GB/s x 6 capacities x 3 policies = 4,608 points of 10,000 requests;
P:617).  Strong scaling (the default for N > 1, SURVEY §8(d) "same point set,
strided sharding"): every N runs the same point set and rank r runs points r, r+N, ...
(no data-path collective; the 384-B summaries are all-gathered once per step, the only
exchange).  `--scaling weak` instead replicates the seed axis N times.  `value` =
simulated request-iterations of all points of all ranks / the max-over-ranks device time
of the K timed steps.

--emulate-ranks G measures the 1..G strong-scaling curve on ONE GPU: each rank's strided
subset runs back to back (ranks share nothing but the final all-gather, so no kernel waits
on another), the curve point is the max-over-ranks step time; beside it the chain floor:
the longest points simulated alone (one warp on one SM), the time no number of GPUs beats.

--impl reference times the CPU oracle (oracle/, the reference arm of this tier) on
the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import numpy as np
import os
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import replace

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import sweep_inputs as si  # noqa: E402

BASE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASE["metric"]
UNIT = "request-iterations/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# Algorithmic work per unit: a request-iteration is an O(1) state update
# of ~10 lane-ops (ctx++, gen++, block-boundary test, finish test, gap, max, last_tok);
# the HBM reference line is the 44 B/request-iteration hot record (read 24 B, write 20 B).
ALG_OPS_PER_UNIT = 10
HBM_BYTES_PER_UNIT = 44
# B200 INT32 ALU peak: MEASURED by tools/alu_peak.cu (profiles/r2/alu_peak.json, 8 independent add
# chains per thread at full occupancy); fallback, if that file is missing, the nominal
# 148 SMs x 128 INT32 lanes x 1965 MHz
ALU_PEAK_PATH = os.path.join(ROOT, "profiles", "r2", "alu_peak.json")


def alu_peak():
    try:
        d = json.load(open(ALU_PEAK_PATH))
        return float(d["int32_peak_gops"]), float(d["warp_issue_peak_gwips"]), \
            "measured: tools/alu_peak.cu INT32 add/xor lane-ops at full occupancy (profiles/r2/alu_peak.json)"
    except Exception:
        return 148 * 128 * 1.965, 148 * 4 * 1.965, "nominal: 148 SMs x 128 lanes x 1965 MHz (no measurement found)"


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def config_for(name: str, world: int, scaling: str = "strong") -> si.SweepConfig:
    """The sweep all ranks run together.  strong: the same point set at every N (C5: the
    65,536-point grid; at N = 1 that is 8 x the per-GPU share).  weak: N copies of the seed axis
    (C5: one seed = 8,192 points per GPU)."""
    if name == "c5":
        cfg = si.c5()
        seeds = list(range(8)) if scaling == "strong" else list(range(world))
        return replace(cfg, workload=replace(cfg.workload, seeds=seeds))
    cfg = si.PRESETS[name]()
    if world > 1 and scaling == "weak":  # replicate the seed axis
        w = cfg.workload
        cfg = replace(cfg, workload=replace(w, seeds=list(range(len(w.seeds) * world))))
    return cfg


WORKLOAD_DESC = {
    "c1": "C1 single simulation: LLaMA-2-7B, A100-like profile, 100 requests at 2 req/s, CONT, 16-token blocks",
    "c2": "C2: LLaMA-2-13B, 1,000 ShareGPT-shaped requests, lambda 1..16 req/s x 8 seeds = 128 points",
    "c3": "C3: LLaMA-2-7B hardware sweep 16 F x 16 B x 6 C x {STATIC, CONT, CONT_RATIO 0.9}, 10k requests, 4,608 points",
    "c4": "C4: LLaMA-2-70B TP 2/4/8 x {CONT, CONT_RATIO 0.9} x {SWAP, RECOMPUTE} x 16 rates x 12 seeds, 10k req, 2,304 points",
    "c5": "C5: 1P:1D pairs 16x16 x {SWAP, RECOMPUTE} x 16 rates x 8 seeds, 10k requests, 65,536 points (weak: one seed = 8,192 points per GPU)",
    # widened rows; measurement only, not BASELINE configs
    "c6": "NEXT-1: P2:D6 node, LLaMA-2-7B, least-outstanding dispatch, {SWAP, RECOMPUTE} x 16 rates x 8 seeds, 10k req, 256 points",
    "c7": "NEXT-2: multi-round conversations + memory cache, LLaMA-2-7B, 2k conversations, {SWAP, RECOMPUTE} x 16 rates x 8 seeds",
    "c8": "NEXT-3: C2 grid x {MIXED, PREFILL_FIRST, CHUNKED 512}, LLaMA-2-13B, 1k requests, 384 points",
    "c9": "NEXT-4: LLaMA-2-70B TP2 SWAP under a 64 MiB preload link, {CONT, CONT_RATIO} x 16 rates x 12 seeds, 10k req",
}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:  # first sample before the timed region
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self, first: int = 0):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        rows = self.rows[first:] or self.rows[-1:]  # samples taken during the timed region
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peaks():
    try:
        return json.load(open(PEAKS_PATH))
    except Exception:
        return {}


# ---------------------------------------------------------------------------- CPU oracle timing
def _oracle_point(args):
    cfg, p = args
    from oracle import oracle as O
    t0 = time.perf_counter()
    r = O.simulate(cfg, p, want=("summary",))
    return r["summary"]["n_request_iterations"], time.perf_counter() - t0


def _noop(x):
    from oracle import oracle as O
    O.lib()
    return x


def oracle_sample(cfg: si.SweepConfig, budget_s: float = 20.0, max_points: int = 64):
    """Run the oracle (as it stands) on a bounded, deterministic sample of the sweep's points,
    one single-threaded process per host core.  Returns (req-it/s, cores, sample desc, RI, wall)."""
    import concurrent.futures as cf
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    P = cfg.num_points
    step = max(1, P // max_points)
    pts = list(range(0, P, step))[:max_points]
    ctx = mp.get_context("spawn")
    ri = 0
    done = 0
    with cf.ProcessPoolExecutor(cores, mp_context=ctx) as ex:
        list(ex.map(_noop, range(cores)))  # start the workers outside the timed region
        t0 = time.perf_counter()
        for b in range(0, len(pts), cores):  # whole batches only: the wall clock covers exactly the work
            for r, _ in ex.map(_oracle_point, [(cfg, p) for p in pts[b:b + cores]]):
                ri += r
                done += 1
            if time.perf_counter() - t0 > budget_s:
                break
        wall = time.perf_counter() - t0
    return ri / wall, cores, f"{done} of {P} points of {cfg.name} (every {step}th point), {cores} processes", ri, wall


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    cfg = config_for(args.config, args.gpus, args.scaling)
    per_step = max(2.0, args.reference_budget / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_sample(cfg, budget_s=per_step)
    vals, ris, walls = [], 0, 0.0
    desc, cores = "", 0
    for _ in range(args.steps):
        v, cores, desc, ri, wall = oracle_sample(cfg, budget_s=per_step)
        ris += ri
        walls += wall
    value = ris / walls
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": walls / args.steps * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int64/f64",
        "data": "synthetic (Philox-seeded Poisson arrivals, SHAREGPT_SYNTH_V1 lengths)",
        "config": {"workload": WORKLOAD_DESC[args.config], "points": cfg.num_points,
                   "sample": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2503_08415_b200 as P

    cfg = config_for(args.config, world, args.scaling)
    sw = P.Sweep(cfg)
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    n_pts = sw.num_points

    def step(gather: bool):
        sw.run(rank, n_pts, world, device=dev, stream=stream)
        if world > 1 and gather:
            with torch.cuda.stream(stream):
                per = -(-n_pts // world) * P.SUMMARY_DTYPE.itemsize
                loc = sw.summaries_device()
                buf = torch.zeros(per, dtype=torch.uint8, device=dev)
                buf[:loc.numel()] = loc
                out = torch.empty(world * per, dtype=torch.uint8, device=dev)
                dist.all_gather_into_tensor(out, buf)
            return out
        return None

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step(True)
    torch.cuda.synchronize(dev)
    # request-iterations of this rank's points (exact: sum of output lengths of finished requests)
    s = sw.summaries()
    ri_local = int(s["n_request_iterations"].sum())
    assert (s["status_flags"] & 16 == 0).all(), "internal error flag set"
    it_max = int(s["n_iterations"].max()) if len(s) else 0  # the longest serial chain
    it_mean = float(s["n_iterations"].mean()) if len(s) else 0.0

    clocks = ClockSampler(local)
    clocks.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sim_ms, wl_ms, sum_ms = [], [], []
    launches = 0
    barrier()
    n_clk0 = len(clocks.rows)
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xff)  # L2 flush between timed steps (not timed)
        starts[i].record(stream)
        step(True)
        ends[i].record(stream)
        info = sw.run_info()  # syncs the stream; reads the per-kernel CUDA events of this step
        sim_ms.append(info["ms_sim"])
        wl_ms.append(info["ms_workload"])
        sum_ms.append(info["ms_summary"])
        launches += info["n_launches"]
    barrier()
    clk = clocks.stop(n_clk0)
    total_ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    t = torch.tensor([total_ms, float(ri_local), sum(sim_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax[0:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tmax[1:2], op=dist.ReduceOp.SUM)
        dist.all_reduce(tmax[2:3], op=dist.ReduceOp.MAX)
        t = tmax
    total_ms, ri_all, sim_ms_max = float(t[0]), int(t[1]), float(t[2])
    value = ri_all * args.steps / (total_ms / 1e3)

    # ---- end to end through the public API with host buffers (create -> run -> D2H summaries)
    e2e_ms = []
    h2d = d2h = 0
    for i in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        sw2 = P.Sweep(cfg)
        sw2.run(rank, n_pts, world, device=dev, stream=stream, workspace=sw._ws)
        host = sw2.summaries()
        if world > 1:
            g = torch.from_numpy(host.view(np.uint8).copy()).to(dev)
            per = -(-n_pts // world) * P.SUMMARY_DTYPE.itemsize
            buf = torch.zeros(per, dtype=torch.uint8, device=dev)
            buf[:g.numel()] = g
            out = torch.empty(world * per, dtype=torch.uint8, device=dev)
            dist.all_gather_into_tensor(out, buf)
            out.cpu()
        info2 = sw2.run_info()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d = info2["h2d_bytes"]
        d2h = host.nbytes
        sw2.close()
    e2e_t = torch.tensor([statistics.median(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = ri_all / (float(e2e_t[0]) / 1e3)

    peaks = measured_peaks()
    alu_gops, issue_gwips, alu_src = alu_peak()
    sim_avg_s = statistics.mean(sim_ms) / 1e3
    achieved_gops = ALG_OPS_PER_UNIT * ri_local / sim_avg_s / 1e9
    hbm_peak = peaks.get("hbm_gbs")
    hbm_src = "MEASURED_PEAKS.json hbm_gbs (measured)"
    if not hbm_peak:  # the profiling guide's fallback when the driver-written file is absent
        hbm_peak, hbm_src = 6650.0, "of fallback: 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"
    hbm_ach = HBM_BYTES_PER_UNIT * ri_local / sim_avg_s / 1e9
    traffic = None
    issue_line = None
    tr_path = os.path.join(ROOT, "profiles", f"dram_{args.config}.json")
    if os.path.exists(tr_path):
        try:
            nc = json.load(open(tr_path))
            traffic = nc.get("dram_bytes_per_launch")
            # SM issue line (supplementary, from the same ncu capture): warp instructions the launch
            # issued / this run's kernel time, against 148 SMs x 4 schedulers x 1 warp-instr/clk
            wi = nc.get("warp_instructions")
            if wi:
                ach = wi / sim_avg_s / 1e9
                pk = issue_gwips
                issue_line = {"warp_instructions_per_launch": wi, "achieved_gwips": ach, "peak_gwips": pk,
                              "frac": ach / pk, "no_instruction_stall_pct": nc.get("no_instruction_stall_pct_of_samples"),
                              "source": "ncu warp instructions of one launch (profiles/dram_<config>.json)"}
        except Exception:
            traffic = None

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            # as the reference arm does: an untimed warm-up pass over the sample, then timed passes
            # (at least two) until the budget -- a single cold pass read ~20% low beside it
            oracle_sample(cfg, budget_s=args.cpu_budget / 4)
            ris = walls = 0.0
            npass = 0
            while npass < 2 or walls < args.cpu_budget / 2:
                _, cores, desc, ri, wall = oracle_sample(cfg, budget_s=args.cpu_budget / 2)
                ris += ri
                walls += wall
                npass += 1
                if npass >= 8:
                    break
            cpu = {"value": ris / walls, "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"{desc}; {npass} timed passes after a warm-up pass"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int64/f64",
            "data": "synthetic (Philox-seeded Poisson arrivals, SHAREGPT_SYNTH_V1 lengths); no trained weights needed",
            "config": {"workload": WORKLOAD_DESC[args.config], "points": n_pts,
                       "points_per_gpu": -(-n_pts // world), "requests_per_point": cfg.workload.num_requests,
                       "request_iterations_per_step": ri_all, "parallelism": f"points sharded p mod {world}",
                       "l2": "flushed (256 MiB write) between timed steps",
                       "step": "workload_kernel + sim_kernel + summary_kernel" + (" + NCCL all-gather" if world > 1 else "")},
            "roofline": {"bound": "alu", "achieved": achieved_gops, "peak": alu_gops, "unit": "Gop/s",
                         "frac": achieved_gops / alu_gops, "traffic": traffic,
                         "kernel": ("sim_node_kernel" if cfg.options.topology == si.PD_PAIR and (cfg.options.pd_prefill + cfg.options.pd_decode > 2 or cfg.options.node_loop) else "sim_kernel"),
                         "kernel_ms": statistics.mean(sim_ms),
                         "per_unit": f"{ALG_OPS_PER_UNIT} lane-ops per request-iteration (SURVEY §8(d))",
                         "peak_source": alu_src,
                         "hbm_line": {"bytes_per_unit": HBM_BYTES_PER_UNIT, "achieved_gbs": hbm_ach,
                                      "peak_gbs": hbm_peak, "frac": (hbm_ach / hbm_peak) if hbm_peak else None,
                                      "peak_source": hbm_src},
                         "issue_line": issue_line,
                         # the serial critical path: iterations of the longest point and the kernel
                         # time per iteration of that chain (one point never splits across warps)
                         "chain": {"max_iterations_per_point": it_max, "mean_iterations_per_point": it_mean,
                                   "ns_per_chain_iteration": statistics.mean(sim_ms) * 1e6 / max(1, it_max)}},
            "kernel_ms": {"workload": statistics.mean(wl_ms), "sim": statistics.mean(sim_ms),
                          "summary": statistics.mean(sum_ms)},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": float(e2e_t[0]), "path": "Sweep(cfg) -> run -> summaries() (C ABI, host buffers)"},
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return 0


def run_emulate(args):
    """Strong-scaling curve on one GPU (VERDICT r1 "Next round #3").  Rank r of G runs points
    p = r (mod G); ranks share nothing but the final 384-B all-gather, so running their subsets
    back to back on one GPU and taking the max-over-ranks step time gives the G-GPU step time
    (minus the all-gather, tens of microseconds over NVLink).  Beside it, the chain floor: each of
    the longest points simulated ALONE (one warp on one SM with its helper warp) -- a point never
    splits across warps or GPUs, so no G beats max over points of that time."""
    import torch
    import paper_2503_08415_b200 as P
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = config_for(args.config, 1, "strong")
    sw = P.Sweep(cfg)
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    n_pts = sw.num_points
    reps = max(1, min(args.steps, 5))

    def timed(begin, end, stride):
        ts = []
        for i in range(reps + 1):  # one warm-up run of this shard
            with torch.cuda.stream(stream):
                flush.fill_(i & 0xff)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sw.run(begin, end, stride, device=dev, stream=stream)
            b.record(stream)
            b.synchronize()
            if i:
                ts.append(a.elapsed_time(b))
        s = sw.summaries()
        return statistics.median(ts), s

    t1, s_all = timed(0, n_pts, 1)
    info1 = sw.run_info()
    ri_total = int(s_all["n_request_iterations"].sum())
    iters = s_all["n_iterations"].astype(np.int64)
    curve = []
    G = 1
    gs = [int(x) for x in args.emulate_gs.split(",")] if args.emulate_gs else None
    while G <= args.emulate_ranks:
        if gs is not None and G not in gs:
            G *= 2
            continue
        per = []
        for r in range(G):
            t, s = (t1, s_all) if G == 1 else timed(r, n_pts, G)
            inf = info1 if G == 1 else sw.run_info()
            per.append({"rank": r, "ms": t, "points": int(len(s)),
                        "request_iterations": int(s["n_request_iterations"].sum()),
                        "max_iterations": int(s["n_iterations"].max()) if len(s) else 0,
                        "helper_mode": inf["helper_mode"], "n_heads": inf["n_heads"],
                        "grid": [inf["sim_blocks"], inf["sim_warps_per_block"]]})
        tmax = max(p["ms"] for p in per)
        curve.append({"gpus": G, "ms_per_step": tmax, "value": ri_total / (tmax / 1e3),
                      "speedup": t1 / tmax, "efficiency": t1 / tmax / G, "ranks": per})
        G *= 2
    # chain floor: the longest points alone
    order = np.argsort(-iters)[:args.floor_points]
    floors = []
    for p in order:
        pt = int(s_all["point"][p])
        t, s = timed(pt, pt + 1, 1)
        floors.append({"point": pt, "iterations": int(iters[p]), "ms_alone": t,
                       "ns_per_iteration": t * 1e6 / max(1, int(iters[p]))})
    floor_ms = max(f["ms_alone"] for f in floors)
    line = {"metric": METRIC, "unit": UNIT, "mode": "emulated strong scaling (one GPU, ranks back to back)",
            "config": {"workload": WORKLOAD_DESC[args.config], "points": n_pts,
                       "request_iterations_per_step": ri_total},
            "curve": curve,
            "chain_floor": {"ms": floor_ms, "value_ceiling": ri_total / (floor_ms / 1e3),
                            "max_speedup_vs_1gpu": t1 / floor_ms, "points": floors,
                            "note": "the longest points simulated alone; no number of GPUs runs a step faster"},
            "gpu": torch.cuda.get_device_name(dev)}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOAD_DESC))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="one GPU: measure the strong-scaling curve for 1, 2, 4, ... G ranks and the chain floor")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--floor-points", type=int, default=4)
    ap.add_argument("--emulate-gs", default="", help="with --emulate-ranks: only these G (comma list)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--reference-budget", type=float, default=120.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("note: --warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.emulate_ranks:
        return run_emulate(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
