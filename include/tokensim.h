/* tokensim.h -- C ABI of the B200-native batched design-space sweep.
 *
 * What this library computes (PAPER.md = arXiv 2503.08415, TokenSim; P:NNN =
 * PAPER.md line): thousands of independent LLM-serving simulations ("points"),
 * one per (hardware profile x scheduling/memory policy x arrival rate x seed).
 * Each point replays TokenSim's worker loop: a workload of requests
 * "generated from datasets and parameters" with Poisson arrivals
 * (reading A24); an iteration-level scheduler invoked at the default
 * end-of-iteration breakpoint doing continuous or static batching
 * with FCFS admission, max-memory-ratio admission (P:460,
 * P:477) and preemption by moving KV to host or recomputing it;
 * a block-granular PagedAttention allocator; a per-operator
 * roofline compute simulator that advances an
 * integer-nanosecond clock; and emits per-request TTFT / TPOT / E2E /
 * normalized / mTPOT latencies and KV memory over
 * time.  The exact semantics are SURVEY.md §8(c) under the
 * readings listed in DESIGN.md; results are bit-identical to oracle/.
 *
 * Execution: every step runs in sm_100a CUDA kernels (workload generation,
 * one persistent warp per point, quantile/summary kernels).  The host side of
 * this library only validates inputs, derives per-profile constants, lays out
 * the workspace and launches.  There is no CPU fallback: without a CUDA device
 * tokensim_sweep_run returns TOKENSIM_E_CUDA.
 *
 * Conventions
 *  - Every call returns a tokensim_status; nothing throws across the ABI.
 *    On failure the message is available from tokensim_last_error().
 *  - Every input struct starts with struct_size = sizeof(struct); a mismatch
 *    is TOKENSIM_E_INVALID (ABI versioning; "unknown keys are errors").
 *  - Pointers are HOST pointers unless the name starts with d_ (DEVICE).
 *  - Ownership: create deep-copies every input (arrays included); the caller
 *    may free its inputs when create returns.  The handle owns its device
 *    tables.  The run workspace is caller-owned device memory (or, if NULL is
 *    passed, handle-owned); it holds the per-point results and must stay alive
 *    until the next run or destroy.  Getters copy into caller buffers; the
 *    two-call pattern applies (out = NULL or capacity = 0 returns *n_out);
 *    a too-small buffer returns TOKENSIM_E_TRUNCATED with *n_out = required.
 *  - A handle is used by one host thread at a time; handles are independent.
 *  - Results do not depend on device, begin/end/stride or the number of GPUs.
 */
#ifndef TOKENSIM_H
#define TOKENSIM_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- status ------------------------------------------------------------ */
typedef enum {
  TOKENSIM_OK = 0,
  TOKENSIM_E_INVALID = -1,   /* validation failed; message names the field path     */
  TOKENSIM_E_NOMEM = -2,     /* host/device allocation failed or workspace too small */
  TOKENSIM_E_CUDA = -3,      /* CUDA error (message carries cudaGetErrorString)      */
  TOKENSIM_E_STATE = -4,     /* call out of order (getter before run, point not run) */
  TOKENSIM_E_RANGE = -5,     /* point / metric / quantile / worker out of range      */
  TOKENSIM_E_TRUNCATED = -6, /* caller buffer too small; *n_out = required count     */
  TOKENSIM_E_OVERFLOW = -7   /* the point's memory trace overflowed its cap          */
} tokensim_status;

/* ---- enums --------------------------------------------------------------- */
enum { TOKENSIM_STATIC = 0, TOKENSIM_CONT = 1, TOKENSIM_CONT_RATIO = 2 };   /* policy.kind   */
enum { TOKENSIM_SWAP = 0, TOKENSIM_RECOMPUTE = 1 };                         /* policy.preempt*/
enum { TOKENSIM_MIXED = 0, TOKENSIM_PREFILL_FIRST = 1, TOKENSIM_CHUNKED = 2 };                    /* policy.iteration_mode */
enum { TOKENSIM_LEN_SHAREGPT_SYNTH_V1 = 0, TOKENSIM_LEN_FIXED = 1, TOKENSIM_LEN_UNIFORM = 2,
       TOKENSIM_LEN_TABLE = 3, TOKENSIM_LEN_TRACE = 4 };                      /* len_dist      */
enum { TOKENSIM_TRACE_NONE = 0, TOKENSIM_TRACE_BINNED = 1, TOKENSIM_TRACE_FULL = 2 };
enum { TOKENSIM_UNIFIED = 0, TOKENSIM_PD_PAIR = 1 };                        /* topology      */
enum { TOKENSIM_LINK_SEQUENTIAL = 0, TOKENSIM_LINK_PRELOAD = 1 };              /* options.link_mode */
enum { TOKENSIM_DISPATCH_ROUND_ROBIN = 0, TOKENSIM_DISPATCH_LEAST_OUTSTANDING = 1,
       TOKENSIM_DISPATCH_LEAST_MEMORY = 2 };                                 /* options.dispatch */
enum { TOKENSIM_TTFT = 0, TOKENSIM_TPOT = 1, TOKENSIM_E2E = 2, TOKENSIM_NORM = 3,
       TOKENSIM_MTPOT = 4 };                                                /* metric        */
enum { TOKENSIM_REQ_UNFINISHED = 0, TOKENSIM_REQ_FINISHED = 1, TOKENSIM_REQ_REJECTED = 2 };
enum { TOKENSIM_PT_TRACE_OVERFLOW = 1, TOKENSIM_PT_ALL_REJECTED = 2, TOKENSIM_PT_HORIZON_HIT = 4,
       TOKENSIM_PT_INTERNAL_ERROR = 16 };                                   /* status_flags  */

/* ---- inputs -------------------------------------------------------------- */
/* Transformer shape.  q = num_heads*head_dim, g = num_kv_heads*head_dim.
 * Weight bytes W and KV bytes per token kvb = 2*L*g*dtype_bytes are derived (SURVEY c.1). */
typedef struct {
  uint32_t struct_size;
  uint32_t num_layers, hidden, num_heads, num_kv_heads, head_dim, ffn_dim, vocab;
  uint32_t dtype_bytes;      /* 2 (fp16)                  */
  uint32_t gated_mlp;        /* 1: up+gate (LLaMA)               */
  uint32_t tied_embeddings;  /* 0                                */
  uint32_t max_model_len;    /* 2048; <= 1<<20                   */
} tokensim_model;

/* Roofline hardware profile.  For tensor parallelism give
 * the AGGREGATE profile (t*F, t*B, t*C) plus tp_degree/tp_link_bw (reading A22). */
typedef struct {
  uint32_t struct_size;
  double peak_flops;          /* FLOP/s, > 0                            */
  double mem_bw;              /* B/s, > 0                               */
  double eff_flops, eff_bw;   /* derating in (0,1] (0.6 / 0.8)   */
  uint64_t mem_capacity;      /* bytes (decimal)                        */
  double reserve_frac;        /* 0.05                           */
  double iter_overhead_s;     /* 200e-6                         */
  double host_link_bw;        /* B/s, swap link (32e9)           */
  uint32_t tp_degree;         /* 1                                      */
  double tp_link_bw;          /* B/s per direction, > 0 if tp_degree>1  */
  uint64_t kv_blocks_override;/* 0 = derive from capacity (tests only)  */
} tokensim_hw;

/* Local scheduler + memory policy. */
typedef struct {
  uint32_t struct_size;
  uint32_t kind;              /* TOKENSIM_STATIC | CONT | CONT_RATIO          */
  uint32_t preempt;           /* TOKENSIM_SWAP | RECOMPUTE                    */
  double max_mem_ratio;       /* CONT_RATIO: (0,1]                    */
  uint32_t max_num_seqs;      /* 256, in [1, 1024]                            */
  uint32_t max_batched_tokens;/* UINT32_MAX = off; else >= max_model_len      */
  uint32_t block_size;        /* 16 tokens                            */
  uint32_t watermark_blocks;  /* 0                                            */
  uint32_t iteration_mode;    /* MIXED: prefills and decodes share an iteration (A3);
                                 PREFILL_FIRST: vLLM v0.6.2 default -- when fresh requests
                                 can be admitted the iteration runs only their prefills
                                 (NEXT-3, reading R-N3); CHUNKED: vLLM chunked prefill --
                                 decodes, then the prefill in progress, resumes and fresh
                                 requests share max_batched_tokens in that order, prompts
                                 split into chunks (P, c0) (NEXT-3, reading R-N3b; needs
                                 max_batched_tokens >= max_num_seqs instead of >=
                                 max_model_len); UNIFIED topology only  */
} tokensim_policy;

/* Bucketed length table: bucket b covers [lo[b], hi[b]); cdf32 holds n_buckets-1 u32
 * thresholds (draw x < cdf32[b]); the last bucket takes the rest. */
typedef struct {
  uint32_t n_buckets;
  const uint32_t *lo, *hi, *cdf32;
} tokensim_len_table;

/* Workload.  rates x seeds are grid axes. */
typedef struct {
  uint32_t struct_size;
  uint32_t num_requests;                /* >= 1 per point                         */
  uint32_t num_rates;
  const double *rates;                  /* req/s, > 0                             */
  uint32_t num_seeds;
  const uint64_t *seeds;
  uint32_t len_dist;                    /* TOKENSIM_LEN_*                         */
  uint32_t prompt_a, prompt_b, output_a, output_b;   /* FIXED: a; UNIFORM: [a,b]  */
  const tokensim_len_table *prompt_table, *output_table;  /* TABLE                */
  const int64_t *trace_arrival_ns;      /* TRACE: non-decreasing, >= 0            */
  const uint32_t *trace_prompt, *trace_output;
  /* NEXT-2 (reading R-N2): num_requests CONVERSATIONS arrive as above
   * (round 0); half have one round, the rest 2..7 (uniform); round r >= 1 arrives an Exp(think
   * mean) gap after round r-1 finishes and its prompt is the prior context plus a new turn drawn
   * like a prompt.  Requests are numbered rid = (rounds of earlier conversations) + r, at most
   * 7 * num_requests per point.  Generated lengths only (not TRACE); UNIFIED topology, MIXED. */
  uint32_t multi_round;
  double think_mean_s;                  /* 5                              */
} tokensim_workload;

typedef struct {
  uint32_t struct_size;
  uint32_t topology;          /* TOKENSIM_UNIFIED | PD_PAIR                          */
  double pd_link_bw;          /* B/s, P->D KV link (200e9)                    */
  uint32_t trace_mode;        /* TOKENSIM_TRACE_NONE | BINNED | FULL                 */
  uint64_t trace_bin_ns;      /* BINNED bin width (1e9)                              */
  uint64_t trace_cap_bytes;   /* per point per worker: BINNED holds 32-B samples; FULL holds
                                 the compressed stream (~4 B per iteration, see
                                 tokensim_get_mem_trace_encoded)                        */
  uint32_t iteration_trace_cap;  /* per point; 0 = off (debug / parity)              */
  double slo_ttft_s;          /* 15                                          */
  double slo_mtpot_s;         /* 0.3                                         */
  int64_t horizon_ns;         /* -1 = run to completion                              */
  uint32_t flags;             /* TOKENSIM_OPT_*; 0 = defaults                        */
  /* NEXT-1: PD_PAIR generalizes to an xP:yD node -- x prefill workers on the
   * prefill profile, y decode workers on the decode profile (x, y >= 1, x + y <= 8; 0 reads
   * as 1) -- with a global scheduler dispatching arrivals to
   * prefill workers and end-of-prefill requests to decode workers (readings R-X1..R-X6). */
  uint32_t pd_prefill_workers;
  uint32_t pd_decode_workers;
  uint32_t dispatch;          /* TOKENSIM_DISPATCH_*; ties go to the lowest worker index    */
  /* NEXT-4: the swap-in link.  SEQUENTIAL (A10): an iteration's swap
   * bytes move before its compute.  PRELOAD: the swap-in streams one layer's chunk at a time
   * through a buffer of preload_buffer_bytes while the layers compute (reading R-N4); never
   * slower than SEQUENTIAL.  The P->D transfer already overlaps both workers (a.9). */
  uint32_t link_mode;         /* TOKENSIM_LINK_SEQUENTIAL | TOKENSIM_LINK_PRELOAD           */
  uint64_t preload_buffer_bytes;  /* PRELOAD: > 0; one chunk fits even if smaller           */
  /* NEXT-2 memory cache: a host LRU cache of conversation contexts.
   * A finishing round stores its context (prompt + output - 1 tokens of KV); admitting a later
   * round of a cached conversation skips that prefix (c.5 prefill row with c0 > 0) and pays
   * cache_fetch_ns_per_block per cached block before its prefill. */
  uint32_t memory_cache;      /* 1 = on (multi-round workloads)                             */
  uint64_t cache_capacity_blocks;  /* 0 = 4 x the point's device KV blocks          */
  double cache_fetch_ns_per_block;  /* 800                                          */
} tokensim_options;
/* options.flags: evaluate quiescent decode stretches one iteration at a time instead of
 * 32 at once (results are identical either way; this exists to prove it). */
enum { TOKENSIM_OPT_NO_FAST_FORWARD = 1,
       /* run a 1P:1D pair through the general xP:yD node loop (results are identical; this
        * exists to prove it) */
       TOKENSIM_OPT_NODE_LOOP = 2 };

/* ---- results ------------------------------------------------------------- */
typedef struct {               /* 32 B; index = request id                         */
  int64_t ttft_ns;             /* first token - arrival (0 if no token yet)        */
  int64_t e2e_ns;              /* finish - arrival (FINISHED only)                 */
  int64_t mtpot_ns;            /* max inter-token gap excluding TTFT (A26)         */
  uint16_t n_preempt;
  uint8_t status;              /* TOKENSIM_REQ_*                                   */
  uint8_t pad;
  uint32_t finish_iter;        /* iteration index k of the finishing iteration     */
} tokensim_request_record;

typedef struct {               /* 32 B                                             */
  int64_t t_ns;                /* FULL: iteration start; BINNED: bin start         */
  int64_t dur_ns;              /* FULL: iteration time T_ns; BINNED: bin width      */
  uint64_t block_ns;           /* integral of blocks-in-use over the sample        */
  uint32_t blocks_max;         /* max blocks in use over the sample                */
  uint32_t n_iter;             /* iterations starting inside the sample            */
} tokensim_mem_sample;

typedef struct {               /* 80 B, debug / parity                             */
  uint64_t k;
  int64_t t_start_ns, T_ns;
  uint32_t n_prefill, n_decode;
  uint64_t N_p, C_d;
  uint32_t n_preempted, n_resumed, n_admitted, n_rejected, n_finished, blocks_in_use;
  uint32_t worker, pad;
} tokensim_iter_record;

typedef struct {               /* 384 B, little-endian; the all-gather payload */
  uint32_t version, status_flags;                                   /*   0 */
  uint64_t point;                                                   /*   8 */
  uint64_t n_requests, n_finished, n_rejected, n_unfinished;        /*  16 */
  uint64_t n_iterations, n_request_iterations, n_preemptions;       /*  48 */
  uint64_t swap_out_bytes, swap_in_bytes;                           /*  72 */
  int64_t first_arrival_ns, last_finish_ns;                         /*  88 */
  uint64_t sched_digest, block_digest, request_digest;              /* 104 */
  uint32_t total_blocks, peak_blocks;                               /* 128 */
  double mean_util;                                                 /* 136 */
  double stat[5][5];  /* [TTFT,TPOT,E2E,NORM,MTPOT][P50,P90,P99,max,mean] s;  144 */
  double throughput_rps, goodput_mtpot_rps, goodput_both_rps;       /* 344 */
  int64_t t_final_ns;                                               /* 368 */
  uint64_t block_ns_sum;                                            /* 376 */
} tokensim_summary;

typedef struct tokensim_sweep tokensim_sweep;   /* opaque handle */

/* ---- lifecycle ----------------------------------------------------------- */
/* Validate, derive per-profile constants (SURVEY c.1) and upload the tables.
 * n_hw profiles x n_pol policies x rates x seeds points (PD_PAIR: n_hw^2 pairs).
 * Errors: E_INVALID (message names the field, e.g.
 * "hw[3].mem_capacity: 20000000000 < weights 13476831232 + reserve ..."), E_NOMEM, E_CUDA.
 * On failure *out = NULL and nothing is leaked. */
tokensim_status tokensim_sweep_create(const tokensim_model *model, const tokensim_hw *hw, uint32_t n_hw,
                                      const tokensim_policy *pol, uint32_t n_pol,
                                      const tokensim_workload *workload, const tokensim_options *options,
                                      tokensim_sweep **out);
/* point = ((hw*n_pol + pol)*n_rates + rate)*n_seeds + seed (row-major grid). */
uint64_t tokensim_sweep_num_points(const tokensim_sweep *h);
/* Device bytes needed to run points begin, begin+stride, ... < end. */
tokensim_status tokensim_sweep_workspace_size(const tokensim_sweep *h, uint64_t begin, uint64_t end,
                                              uint64_t stride, size_t *bytes);
/* Enqueue the whole sweep on cuda_stream (a cudaStream_t; NULL = legacy default stream) on
 * `device`: workload generation -> persistent simulation kernel -> quantile/summary kernel.
 * d_workspace: >= workspace_size bytes of device memory, 256-B aligned, or NULL for a
 * handle-owned allocation.  Asynchronous: results are valid after the stream completes
 * (getters synchronize).  Errors: E_RANGE (bad range), E_NOMEM (workspace too small), E_CUDA. */
tokensim_status tokensim_sweep_run(tokensim_sweep *h, int device, uint64_t begin, uint64_t end,
                                   uint64_t stride, void *d_workspace, size_t ws_bytes,
                                   void *cuda_stream);
/* Number of points run by the last tokensim_sweep_run. */
uint64_t tokensim_sweep_num_run(const tokensim_sweep *h);

/* ---- results ------------------------------------------------------------- */
/* Exact nearest-rank quantiles (rank = max(1, ceil(q_bp*n/10^4))) of
 * `metric` over the point's finished requests, in seconds (0 if no sample).  q_bp in
 * [0, 10000].  Computed by a GPU select kernel over the point's records.  For points this
 * process did not run, only q_bp in {5000, 9000, 9900, 10000} are served, from summaries
 * imported with tokensim_import_summaries; anything else is E_STATE. */
tokensim_status tokensim_get_latency_quantiles(const tokensim_sweep *h, uint64_t point, uint32_t metric,
                                               const uint32_t *q_bp, uint32_t n_q, double *out_seconds);
/* KV memory over time of one worker: 0 = unified; PD_PAIR: prefill workers
 * 0..x-1, decode workers x..x+y-1 (1P:1D: 0 = prefill, 1 = decode).  E_RANGE for any other
 * worker.  Returns E_OVERFLOW (with the samples that fit) if the trace hit its cap.  FULL
 * traces are stored compressed on the device and decoded here (one sample per iteration:
 * t_ns = start, dur_ns = T, block_ns = blocks * T, blocks_max = blocks, n_iter = 1). */
tokensim_status tokensim_get_mem_trace(const tokensim_sweep *h, uint64_t point, uint32_t worker,
                                       tokensim_mem_sample *out, uint64_t capacity, uint64_t *n_out);
/* The FULL trace as stored: a byte stream (SURVEY §8(a.8) "delta + varint"; reading A28, one
 * record per iteration k) of three unsigned LEB128 varints per iteration,
 *     t_start_k - t_end_{k-1}  (>= 0),  zigzag(T_k - T_{k-1}),  zigzag(blocks_k - blocks_{k-1}),
 * with t_end_{-1} = T_{-1} = blocks_{-1} = 0 and zigzag(v) = (v << 1) ^ (v >> 63).  The
 * stream holds whole records only: one that would cross trace_cap_bytes ends it (E_OVERFLOW).
 * *n_bytes = stream length, *n_samples = its iterations; out = NULL or capacity = 0 only
 * queries them; a smaller buffer is E_TRUNCATED.  E_STATE unless trace_mode = FULL. */
tokensim_status tokensim_get_mem_trace_encoded(const tokensim_sweep *h, uint64_t point, uint32_t worker,
                                               uint8_t *out, uint64_t capacity, uint64_t *n_bytes,
                                               uint64_t *n_samples);
tokensim_status tokensim_get_summary(const tokensim_sweep *h, uint64_t point, tokensim_summary *out);
/* All summaries of the last run, in run order (point begin, begin+stride, ...). */
tokensim_status tokensim_get_summaries(const tokensim_sweep *h, tokensim_summary *out, uint64_t capacity,
                                       uint64_t *n_out);
/* Device pointer to the last run's summaries (n_run x 384 B) for an all-gather. */
tokensim_status tokensim_get_summaries_device(const tokensim_sweep *h, const void **d_ptr, size_t *bytes);
/* Install summaries of points run elsewhere (after the all-gather); each record carries
 * its point index.  bytes must be a multiple of 384. */
tokensim_status tokensim_import_summaries(tokensim_sweep *h, const void *host_ptr, size_t bytes);
tokensim_status tokensim_get_request_records(const tokensim_sweep *h, uint64_t point,
                                             tokensim_request_record *out, uint64_t capacity, uint64_t *n_out);
/* Per-iteration schedule trace (debug/parity; needs options.iteration_trace_cap > 0). */
tokensim_status tokensim_get_iteration_trace(const tokensim_sweep *h, uint64_t point,
                                             tokensim_iter_record *out, uint64_t capacity, uint64_t *n_out);
/* Per-point workload the kernels generated (group of the point's rate and seed). */
tokensim_status tokensim_get_workload(const tokensim_sweep *h, uint64_t point, int64_t *arrival_ns,
                                      uint32_t *prompt, uint32_t *output, uint64_t capacity);

/* Launch facts of the last run: per-kernel device times from CUDA events recorded on the
 * run's stream (valid once the stream has completed; this call synchronizes), the launch
 * geometry of the simulation kernel, and the host->device bytes the run copied. */
typedef struct {
  double ms_workload, ms_sim, ms_summary;   /* kernel durations, milliseconds          */
  uint32_t n_launches;                      /* kernels this library launched in the run */
  uint32_t sim_blocks, sim_warps_per_block; /* persistent grid                          */
  uint32_t smem_per_warp;                   /* bytes of shared memory per point/warp    */
  uint64_t n_run;                           /* points run                               */
  uint64_t h2d_bytes;                       /* tables (first run on a device) + order   */
  uint64_t workspace_bytes;
  uint32_t helper_mode;                     /* one point per CTA with a helper warp: 1 with
                                               extended stretches, 2 without; 0: 8 warps/SM */
  uint32_t n_heads;                         /* longest points given an SM of their own      */
} tokensim_run_info;
tokensim_status tokensim_get_run_info(const tokensim_sweep *h, tokensim_run_info *out);

/* Per-point execution profile of the last run (observability): iterations simulated, how
 * many of them were committed by time-parallel fast-forward stretches, and SM cycles.
 * sm_cycles is always measured.  The path/phase cycle splits and ff_failed / ff_cut are
 * compiled out of the product library (they cost 5-10% of the simulation kernel) and read 0
 * unless the library was built with -DTS_PROFILE=1 (libtokensim_prof.so, tools/prof_run.py). */
typedef struct {
  uint64_t n_iterations, ff_iterations, ff_stretches, sm_cycles;
  uint64_t cycles_ff, cycles_ff_failed, cycles_normal;  /* split of sm_cycles by path */
  uint64_t stretch_phase_cycles[8];  /* inside successful stretches: scan of R / cost + cut /
                                        block allocation / slot updates + finishes / digests /
                                        memory trace / compaction / bookkeeping.  xP:yD node
                                        points instead: epochs / scheduler-phase cycles (warp 0)
                                        / warp 0's decode-phase cycles / the largest and the
                                        summed decode-phase cycles over decode warps / warp 0's
                                        horizon computations / its waits for the slowest decode
                                        warp / 0 (the product build measures these too)     */
  uint64_t n_transfers, transfer_bytes;  /* PD_PAIR: P->D KV transfers started and their bytes */
  uint64_t normal_phase_cycles[8];  /* normal iterations: reservation+preemption / resume /
                                       admission / block allocation / cost / commit pass /
                                       compaction / digests+trace                           */
  uint64_t ff_failed[5];  /* unified worker: fast-forward attempts that did not run (< 2
                             iterations), by what stopped them: an admission/resume was possible /
                             memory / the next arrival / the blocked head unblocks / other */
  uint64_t ff_cut[5];     /* what ended each stretch: memory / a finishing request / the next
                             arrival / the blocked head / 32 iterations or other */
} tokensim_point_profile;
tokensim_status tokensim_get_point_profile(const tokensim_sweep *h, uint64_t point, tokensim_point_profile *out);

/* Environment variables read by tokensim_sweep_run -- A/B experiments only; results never
 * depend on them (every kernel variant and queue order gives the same bytes), only the launch
 * choice and the order of the point queue do.  Unset = the measured defaults.
 *   TOKENSIM_HELPER=0|1    helper-warp kernel (lean or full) off / on regardless of points per SM
 *   TOKENSIM_XS=0|1        helper kernel without / with extended stretches
 *   TOKENSIM_WPB=n         simulating warps per CTA (1..4) of the independent-warp kernel (default 4,
 *                          or 3 x 2 CTAs per SM for a lean run of 4-8 points per SM)
 *   TOKENSIM_BPS=n         at most n CTAs per SM
 *   TOKENSIM_HEADS=K       helper kernel: the K longest-estimated points get an SM each
 *   TOKENSIM_NODE_TWO=0|1  xP:yD node kernel: one CTA per SM / the 168-register build, two
 *                          per SM (default: two once there are more points than SMs)
 *   TOKENSIM_NODE_SW=0|1   xP:yD node kernel: the scheduler on a warp of its own (default: when the
 *                          points fit one CTA per SM and the two-per-SM build is not used)
 *   TOKENSIM_LPT_OLD=1     order the queue by span / T(1) (round 1) instead of the cost sketch
 *   TOKENSIM_LPT_HELPER=1|2  helper runs: order by the sketch's iterations / cost
 *   TOKENSIM_LPT_COSTS=path  order by per-point costs read from `path` (n_points doubles)
 *   TOKENSIM_DEBUG_XS=1    print the median point's quiet-stretch estimate (extended-stretch choice)
 *   TOKENSIM_LPT_DUMP=path write the queue-order cost estimates (one double per run point) */

/* Message of the last failing call on h (NULL: the calling thread's last create error). */
const char *tokensim_last_error(const tokensim_sweep *h);
void tokensim_sweep_destroy(tokensim_sweep *h);

/* Library/kernel version string, e.g. "tokensim-b200 1 sm_100a". */
const char *tokensim_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TOKENSIM_H */
