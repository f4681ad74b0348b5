"""Seeded, synthetic sweep inputs shared by the oracle and the CUDA path.

This module is the ONLY code both sides may import.  It holds configuration
data (model shapes, hardware grids, policies, arrival rates, seeds, the
synthetic length table) and nothing of the method's arithmetic: no Philox,
no log, no cost model, no derived constants.  Each side derives everything
else itself from these plain values.

Citations: ``P:NNN`` = /root/reference/PAPER.md line, ``S:NNN`` = SPEC.md line
(the reference tree is not present on the GPU box; citations are text only).
Config presets follow SURVEY.md §8(d) ("Concrete configs") and BASELINE.json
``configs``.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence

UINT32_MAX = 0xFFFFFFFF

# ---------------------------------------------------------------- model shapes
@dataclass(frozen=True)
class Model:
    """Transformer shape.  LLaMA-2 shapes are public model-card
    facts (reading A30)."""
    name: str
    num_layers: int
    hidden: int
    num_heads: int
    num_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab: int
    dtype_bytes: int = 2          # fp16
    gated_mlp: int = 1
    tied_embeddings: int = 0
    max_model_len: int = 2048


LLAMA2_7B = Model("llama-2-7b", 32, 4096, 32, 32, 128, 11008, 32000)
LLAMA2_13B = Model("llama-2-13b", 40, 5120, 40, 40, 128, 13824, 32000)
LLAMA2_70B = Model("llama-2-70b", 80, 8192, 64, 8, 128, 28672, 32000)

# ---------------------------------------------------------------- hardware
@dataclass(frozen=True)
class Hw:
    """Roofline hardware profile."""
    peak_flops: float = 312e12      # A100 fp16
    mem_bw: float = 2.039e12        # A100-80GB (reading A32)
    mem_capacity: int = 80_000_000_000
    eff_flops: float = 0.6          # S:242 (uncalibrated default, A21)
    eff_bw: float = 0.8
    reserve_frac: float = 0.05
    iter_overhead_s: float = 200e-6
    host_link_bw: float = 32e9
    tp_degree: int = 1
    tp_link_bw: float = 0.0
    kv_blocks_override: int = 0     # tests only


A100 = Hw()
# closed-form test profile: eff = 1, overhead 0 (SURVEY §8 c.5 "verified" rows)
A100_IDEAL = Hw(eff_flops=1.0, eff_bw=1.0, iter_overhead_s=0.0)

# ---------------------------------------------------------------- policies
STATIC, CONT, CONT_RATIO = "static", "cont", "cont_ratio"
SWAP, RECOMPUTE = "swap", "recompute"
MIXED, PREFILL_FIRST, CHUNKED = "mixed", "prefill_first", "chunked"
ROUND_ROBIN, LEAST_OUTSTANDING, LEAST_MEMORY = "round_robin", "least_outstanding", "least_memory"
SEQUENTIAL, PRELOAD = "sequential", "preload"


@dataclass(frozen=True)
class Policy:
    """Local-scheduler + memory policy."""
    kind: str = CONT
    preempt: str = SWAP
    max_mem_ratio: float = 1.0
    max_num_seqs: int = 256
    max_batched_tokens: int = UINT32_MAX
    block_size: int = 16
    watermark_blocks: int = 0
    iteration_mode: str = MIXED     # MIXED (A3) | PREFILL_FIRST (vLLM v0.6.2 default) | CHUNKED (NEXT-3)


# ---------------------------------------------------------------- workload
@dataclass(frozen=True)
class LenTable:
    """Bucketed length table: bucket b covers [lo[b], hi[b]); thr holds the
    n-1 u32 thresholds (the last bucket takes the rest)."""
    lo: Sequence[int]
    hi: Sequence[int]
    thr: Sequence[int]


# SHAREGPT_SYNTH_V1 (reading A25).  Thresholds are normative.
SHAREGPT_PROMPT = LenTable(
    lo=(4, 16, 32, 64, 128, 256, 512),
    hi=(16, 32, 64, 128, 256, 512, 1024),
    thr=(644245094, 1309965025, 2040109466, 2770253906, 3457448673, 3994319585),
)
SHAREGPT_OUTPUT = LenTable(
    lo=(4, 16, 32, 64, 128, 256, 512, 1024),
    hi=(16, 32, 64, 128, 256, 512, 1024, 2048),
    thr=(429496730, 773094113, 1159641170, 1717986918, 2448131359, 3307124818,
         4101693768),
)

FIXED, UNIFORM, TABLE, TRACE = "fixed", "uniform", "table", "trace"


@dataclass(frozen=True)
class Workload:
    """Request stream description.  Rates x seeds form the
    workload axes of the grid."""
    num_requests: int
    rates: Sequence[float]
    seeds: Sequence[int]
    len_dist: str = TABLE
    prompt_a: int = 0
    prompt_b: int = 0
    output_a: int = 0
    output_b: int = 0
    prompt_table: Optional[LenTable] = SHAREGPT_PROMPT
    output_table: Optional[LenTable] = SHAREGPT_OUTPUT
    trace_arrival_ns: Optional[Sequence[int]] = None
    trace_prompt: Optional[Sequence[int]] = None
    trace_output: Optional[Sequence[int]] = None
    multi_round: bool = False          # NEXT-2: num_requests conversations of 1..7 rounds
    think_mean_s: float = 5.0          # NEXT-2: mean think time between rounds


NONE_TRACE, BINNED, FULL = "none", "binned", "full"
UNIFIED, PD_PAIR = "unified", "pd_pair"


@dataclass(frozen=True)
class Options:
    topology: str = UNIFIED
    pd_link_bw: float = 200e9
    trace_mode: str = BINNED
    trace_bin_ns: int = 1_000_000_000
    trace_cap_bytes: int = 1 << 20
    iteration_trace_cap: int = 0
    slo_ttft_s: float = 15.0
    slo_mtpot_s: float = 0.3
    horizon_ns: int = -1
    fast_forward: bool = True          # CUDA path only: time-parallel quiescent stretches
    pd_prefill: int = 1                # PD: prefill workers x (NEXT-1 xP:yD node; x + y <= 8)
    pd_decode: int = 1                 # PD: decode workers y
    dispatch: str = "round_robin"      # global scheduler: ROUND_ROBIN | LEAST_OUTSTANDING | LEAST_MEMORY
    node_loop: bool = False            # CUDA path only: run a 1P:1D pair through the xP:yD loop
    link_mode: str = "sequential"      # swap-in link: SEQUENTIAL (A10) | PRELOAD (NEXT-4)
    memory_cache: bool = False         # NEXT-2: host KV cache of conversation contexts
    cache_capacity_blocks: int = 0     # 0 = 4x the device KV blocks
    cache_fetch_ns_per_block: float = 800.0
    preload_buffer_bytes: int = 1 << 30  # PRELOAD buffer


@dataclass(frozen=True)
class SweepConfig:
    name: str
    model: Model
    hws: Sequence[Hw]
    policies: Sequence[Policy]
    workload: Workload
    options: Options = field(default_factory=Options)

    @property
    def num_points(self) -> int:
        n_hw = len(self.hws)
        if self.options.topology == PD_PAIR:
            n_hw = n_hw * n_hw
        return n_hw * len(self.policies) * len(self.workload.rates) * len(self.workload.seeds)

    def point_coords(self, point: int):
        """Row-major grid decode: point = ((hw*n_pol + pol)*n_rates + rate)*n_seeds + seed
        (SURVEY §8(b) "Point grid")."""
        ns, nr, npol = len(self.workload.seeds), len(self.workload.rates), len(self.policies)
        seed = point % ns
        point //= ns
        rate = point % nr
        point //= nr
        pol = point % npol
        hw = point // npol
        return hw, pol, rate, seed


# ---------------------------------------------------------------- presets
def c1() -> SweepConfig:
    """BASELINE configs[0]: one LLaMA-7B point, A100-like, 100 requests at 2 req/s."""
    return SweepConfig("c1", LLAMA2_7B, [A100], [Policy()],
                       Workload(100, [2.0], [0]))


def c2(n_seeds: int = 8) -> SweepConfig:
    """BASELINE configs[1]: LLaMA-2-13B, 1,000 requests, lambda in 1..16 x seeds 0..7."""
    return SweepConfig("c2", LLAMA2_13B, [A100], [Policy()],
                       Workload(1000, [float(r) for r in range(1, 17)], list(range(n_seeds))))


def c3_hws() -> List[Hw]:
    out = []
    for kf in range(-9, 7):
        for kb in range(-9, 7):
            for cap in (20, 40, 80, 160, 320, 640):
                out.append(Hw(peak_flops=312e12 * 2.0 ** (kf / 3.0),
                              mem_bw=2.039e12 * 2.0 ** (kb / 3.0),
                              mem_capacity=cap * 1_000_000_000))
    return out


def c3() -> SweepConfig:
    """BASELINE configs[2]: 16x16x6 hardware grid x {STATIC, CONT, CONT_RATIO 0.9},
    LLaMA-7B, 10k requests at 4 req/s (4,608 points >= 4,096)."""
    pols = [Policy(kind=STATIC), Policy(kind=CONT), Policy(kind=CONT_RATIO, max_mem_ratio=0.9)]
    return SweepConfig("c3", LLAMA2_7B, c3_hws(), pols, Workload(10_000, [4.0], [0]))


def c4_hws() -> List[Hw]:
    return [Hw(peak_flops=t * 312e12, mem_bw=t * 2.039e12, mem_capacity=t * 80_000_000_000,
               tp_degree=t, tp_link_bw=300e9) for t in (2, 4, 8)]


def c4() -> SweepConfig:
    """BASELINE configs[3]: LLaMA-70B on TP 2/4/8 aggregate profiles, {CONT, CONT_RATIO 0.9}
    x {SWAP, RECOMPUTE}, lambda = 0.5*2^(k/4), seeds 0..11 (2,304 points >= 2,048)."""
    pols = [Policy(kind=k, preempt=pm, max_mem_ratio=r)
            for (k, r) in ((CONT, 1.0), (CONT_RATIO, 0.9)) for pm in (SWAP, RECOMPUTE)]
    rates = [0.5 * 2.0 ** (k / 4.0) for k in range(16)]
    return SweepConfig("c4", LLAMA2_70B, c4_hws(), pols, Workload(10_000, rates, list(range(12))))


def c5_hws() -> List[Hw]:
    return [Hw(peak_flops=312e12 * fs, mem_bw=2.039e12 * bs)
            for fs in (0.25, 0.5, 1.0, 2.0) for bs in (0.5, 1.0, 2.0, 4.0)]


def c5() -> SweepConfig:
    """BASELINE configs[4]: 1P:1D pairs over a 4x4 profile grid (16x16 pairs) x
    {SWAP, RECOMPUTE} x 16 rates x 8 seeds = 65,536 points."""
    pols = [Policy(preempt=SWAP), Policy(preempt=RECOMPUTE)]
    rates = [0.5 * 2.0 ** (k / 4.0) for k in range(16)]
    return SweepConfig("c5", LLAMA2_7B, c5_hws(), pols, Workload(10_000, rates, list(range(8))),
                       Options(topology=PD_PAIR))


# ---- sweeps for the SURVEY §8(f) rows (measurement of each widened row; not BASELINE configs)
def c6() -> SweepConfig:
    """NEXT-1: one 8-GPU node as P2:D6 (fig:pd shape), LLaMA-2-7B on A100-like workers,
    least-outstanding dispatch, {SWAP, RECOMPUTE} x 16 rates (3 x 2^(k/4) req/s) x 8 seeds,
    10k requests: 256 points."""
    pols = [Policy(preempt=SWAP), Policy(preempt=RECOMPUTE)]
    rates = [3.0 * 2.0 ** (k / 4.0) for k in range(16)]
    return SweepConfig("c6", LLAMA2_7B, [A100], pols, Workload(10_000, rates, list(range(8))),
                       Options(topology=PD_PAIR, pd_prefill=2, pd_decode=6, dispatch=LEAST_OUTSTANDING))


def c7() -> SweepConfig:
    """NEXT-2: multi-round conversations with the host memory cache (Finding 6 shape),
    LLaMA-2-7B, 2,000 conversations (half single-round, else 2..7 rounds, 5 s think time),
    CONT x {SWAP, RECOMPUTE} x 16 rates (0.5 x 2^(k/4)) x 8 seeds: 256 points."""
    pols = [Policy(preempt=SWAP), Policy(preempt=RECOMPUTE)]
    rates = [0.5 * 2.0 ** (k / 4.0) for k in range(16)]
    return SweepConfig("c7", LLAMA2_7B, [A100], pols,
                       Workload(2_000, rates, list(range(8)), multi_round=True, think_mean_s=5.0),
                       Options(memory_cache=True))


def c8() -> SweepConfig:
    """NEXT-3: the C2 grid under {MIXED, PREFILL_FIRST, CHUNKED (512-token budget)} iterations:
    384 points."""
    pols = [Policy(), Policy(iteration_mode=PREFILL_FIRST), Policy(iteration_mode=CHUNKED, max_batched_tokens=512)]
    return SweepConfig("c8", LLAMA2_13B, [A100], pols, Workload(1000, [float(r) for r in range(1, 17)], list(range(8))))


def c9() -> SweepConfig:
    """NEXT-4: C4's preemption-heavy TP2 profile with SWAP under a 64 MiB preload link,
    {CONT, CONT_RATIO 0.9} x 16 rates x 12 seeds, 10k requests: 384 points."""
    pols = [Policy(kind=k, preempt=SWAP, max_mem_ratio=r) for (k, r) in ((CONT, 1.0), (CONT_RATIO, 0.9))]
    rates = [0.5 * 2.0 ** (k / 4.0) for k in range(16)]
    return SweepConfig("c9", LLAMA2_70B, c4_hws()[:1], pols, Workload(10_000, rates, list(range(12))),
                       Options(link_mode=PRELOAD, preload_buffer_bytes=64 << 20))


PRESETS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5, "c6": c6, "c7": c7, "c8": c8, "c9": c9}


def with_requests(cfg: SweepConfig, n: int) -> SweepConfig:
    return replace(cfg, workload=replace(cfg.workload, num_requests=n))


def subset(cfg: SweepConfig, hws=None, policies=None, rates=None, seeds=None) -> SweepConfig:
    """Restrict grid axes (index lists) -- used to build small parity cases."""
    w = cfg.workload
    return replace(
        cfg,
        hws=[cfg.hws[i] for i in hws] if hws is not None else cfg.hws,
        policies=[cfg.policies[i] for i in policies] if policies is not None else cfg.policies,
        workload=replace(
            w,
            rates=[w.rates[i] for i in rates] if rates is not None else w.rates,
            seeds=[w.seeds[i] for i in seeds] if seeds is not None else w.seeds,
        ),
    )
