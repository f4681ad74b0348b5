/* oracle.h -- C ABI of the CPU ORACLE (test infrastructure only).
 *
 * This header belongs to oracle/ alone.  It shares nothing with include/ or
 * the CUDA path: the structs below are the oracle's own, and only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load liboracle.so.
 *
 * One call simulates ONE sweep point, sequentially, following SURVEY.md §8(c)
 * (c.1-c.6) under the readings listed in DESIGN.md.  PAPER.md citations
 * (P:NNN) are given where the paper defines the step.
 */
#ifndef TOKENSIM_ORACLE_H
#define TOKENSIM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { OR_STATIC = 0, OR_CONT = 1, OR_CONT_RATIO = 2 };
enum { OR_SWAP = 0, OR_RECOMPUTE = 1 };
enum { OR_LEN_FIXED = 1, OR_LEN_UNIFORM = 2, OR_LEN_TABLE = 3, OR_LEN_TRACE = 4 };
enum { OR_TRACE_NONE = 0, OR_TRACE_BINNED = 1, OR_TRACE_FULL = 2 };
enum { OR_UNIFIED = 0, OR_PD_PAIR = 1 };
enum { OR_MIXED = 0, OR_PREFILL_FIRST = 1, OR_CHUNKED = 2 };
enum { OR_DISPATCH_RR = 0, OR_DISPATCH_LEAST_OUTSTANDING = 1, OR_DISPATCH_LEAST_MEMORY = 2 };
enum { OR_MAX_WORKERS = 8 };
enum { OR_LINK_SEQUENTIAL = 0, OR_LINK_PRELOAD = 1 };

typedef struct {
  /* model */
  uint32_t L, h, n_heads, n_kv, head_dim, ffn, vocab, dtype_bytes, gated, tied, max_model_len;
  /* hardware profile; for PD_PAIR this is the PREFILL worker */
  double peak_flops, mem_bw, eff_flops, eff_bw;
  uint64_t mem_capacity;
  double reserve_frac, iter_overhead_s, host_link_bw;
  uint32_t tp_degree;
  double tp_link_bw;
  uint64_t kv_blocks_override;
  /* second profile: the DECODE worker (PD_PAIR only) */
  double d_peak_flops, d_mem_bw, d_eff_flops, d_eff_bw;
  uint64_t d_mem_capacity;
  double d_reserve_frac, d_iter_overhead_s, d_host_link_bw;
  uint32_t d_tp_degree;
  double d_tp_link_bw;
  uint64_t d_kv_blocks_override;
  /* policy */
  uint32_t kind, preempt;
  double max_mem_ratio;
  uint32_t max_num_seqs, max_batched_tokens, block_size, watermark_blocks;
  /* workload */
  uint32_t num_requests;
  double rate;
  uint64_t seed;
  uint32_t len_dist, prompt_a, prompt_b, output_a, output_b;
  uint32_t pt_n;
  const uint32_t *pt_lo, *pt_hi, *pt_thr;
  uint32_t ot_n;
  const uint32_t *ot_lo, *ot_hi, *ot_thr;
  const int64_t *trace_arrival_ns;
  const uint32_t *trace_prompt, *trace_output;
  /* options */
  uint32_t topology;
  double pd_link_bw;
  uint32_t trace_mode;
  uint64_t trace_bin_ns, trace_cap_samples;
  double slo_ttft_s, slo_mtpot_s;
  int64_t horizon_ns;
  uint32_t check_invariants;   /* 1: assert c.8 invariants every iteration */
  uint32_t keep_events;        /* 1: keep the block event log              */
  uint32_t iter_mode;          /* OR_MIXED (A3) | OR_PREFILL_FIRST | OR_CHUNKED (NEXT-3) */
  /* NEXT-1 xP:yD node (PD_PAIR topology): x prefill + y decode workers, x + y <= 8 */
  uint32_t n_prefill, n_decode;  /* 0 reads as 1 */
  uint32_t dispatch;             /* OR_DISPATCH_* (global scheduler) */
  uint32_t force_general;        /* 1: run the x:y loop even for 1:1 (pins it to the 1:1 loop) */
  /* NEXT-4 communication model: swap-in link mode and buffer */
  uint32_t link_mode;            /* OR_LINK_SEQUENTIAL | OR_LINK_PRELOAD */
  uint64_t preload_buffer_bytes;
  /* NEXT-2 multi-round conversations and host memory cache */
  uint32_t multi_round;          /* num_requests = conversations of 1..7 rounds */
  double think_mean_s;
  uint32_t memory_cache;         /* 1: hits skip the cached prefix at 800 ns/block */
  uint64_t cache_capacity_blocks;  /* 0 = 4x device KV blocks */
  double cache_fetch_ns_per_block;
} oracle_cfg;

typedef struct {
  uint64_t W, kvb, block_bytes, reserve, total_blocks, ratio_limit;
  double invF, invB, invH, invT, scale_ns;
  int64_t slo_ttft_ns, slo_mtpot_ns;
} oracle_derived;

typedef struct {
  int64_t ttft_ns, e2e_ns, mtpot_ns;
  uint32_t n_preempt, status; /* 0 unfinished, 1 finished, 2 rejected */
  uint64_t finish_k;
} oracle_record;

typedef struct {
  uint64_t k;
  int64_t t_start, T_ns;
  uint64_t S_p, D, N_p, C_d, m, n_resumed, n_admitted, n_rejected, n_finished, blocks;
  uint32_t worker; /* 0 unified; PD: prefill workers 0..x-1, decode workers x..x+y-1 */
  uint32_t pad;
} oracle_iter;

typedef struct {
  int64_t t_ns, dur_ns;
  uint64_t block_ns;
  uint32_t blocks_max, n_iter;
} oracle_sample;

typedef struct {
  uint64_t k;
  uint32_t kind, req, block, worker;
} oracle_event;

typedef struct {
  uint32_t status_flags; /* 1 trace overflow, 2 all rejected, 4 horizon hit */
  uint64_t n_requests, n_finished, n_rejected, n_unfinished;
  uint64_t n_iterations, n_request_iterations, n_preemptions, swap_out_bytes, swap_in_bytes;
  int64_t first_arrival_ns, last_finish_ns, t_final;
  uint64_t sched_digest, block_digest, request_digest;
  uint64_t total_blocks, peak_blocks, block_ns_sum;
  double mean_util;
  double stat[5][5]; /* [TTFT,TPOT,E2E,NORM,MTPOT][P50,P90,P99,max,mean] seconds */
  double throughput_rps, goodput_mtpot_rps, goodput_both_rps;
  uint64_t n_transfers, transfer_bytes; /* PD_PAIR only */
} oracle_summary;

typedef struct oracle_run oracle_run;

/* ---- unit functions used by the pin tests ---- */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double oracle_det_log(double u);
/* returns 0, or -1 with a message from oracle_error() */
int oracle_derive(const oracle_cfg *cfg, int decode_worker, oracle_derived *out);
int oracle_workload(const oracle_cfg *cfg, int64_t *arrival, uint32_t *prompt, uint32_t *output);
/* iteration time of one explicit batch (c.5): prefill entries (P[i], c0[i]) -- emits[i] = 0 marks
   a non-final chunk without an LM-head row (NULL: all emit) -- and decode contexts c[j] */
int64_t oracle_iter_time_ns(const oracle_cfg *cfg, int decode_worker, uint32_t n_prefill,
                            const uint32_t *P, const uint32_t *c0, const uint32_t *emits,
                            uint32_t n_decode, const uint32_t *c, uint64_t swap_out, uint64_t swap_in);
/* NEXT-4: completion time of an n-chunk preload pipeline (load a, consume b, `slots` buffer
   chunks) -- the consumer's finish of the last chunk */
double oracle_pipeline(uint64_t n_chunks, double a, double b, uint64_t slots);
uint64_t oracle_fold(const uint64_t *fields, uint32_t n);

/* NEXT-2: the multi-round workload of one point -- per request (conversation c, round r) in id
   order rid = base_c + r: round-0 arrival (r = 0) or think gap (r >= 1), prompt, output, conv.
   Returns the number of requests (<= 7 * num_requests), or -1. */
int64_t oracle_workload_rounds(const oracle_cfg *cfg, int64_t *arrival_or_think, uint32_t *prompt,
                               uint32_t *output, uint32_t *conv);

/* ---- one point, start to finish ---- */
oracle_run *oracle_simulate(const oracle_cfg *cfg);      /* NULL on error */
const char *oracle_error(void);
void oracle_summary_get(const oracle_run *r, oracle_summary *out);
uint64_t oracle_records(const oracle_run *r, oracle_record *out);   /* out may be NULL */
uint64_t oracle_iters(const oracle_run *r, oracle_iter *out);
uint64_t oracle_trace(const oracle_run *r, int worker, oracle_sample *out);  /* worker < x + y */
uint64_t oracle_events(const oracle_run *r, oracle_event *out);
void oracle_free(oracle_run *r);

#ifdef __cplusplus
}
#endif
#endif
