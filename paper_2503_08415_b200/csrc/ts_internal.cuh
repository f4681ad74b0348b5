// ts_internal.cuh -- device-side data layout shared by the kernels and the host runtime.
// Nothing here is shared with oracle/ (the oracle has its own structs and code).
#pragma once
#include <cstdlib>
#include <cstddef>
#include <cstdint>

#include "../../include/tokensim.h"

namespace ts {

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;

// Model constants (SURVEY c.5 notation), all exact integers.
struct DevModel {
  u64 L, h, q, g, f, fu, V, s;
  u64 q2g;     // q + 2g
  u64 hq2g;    // h*(q+2g)
  u64 qh;      // q*h
  u64 hfu;     // h*f_u
  u64 fh;      // f*h
  u64 Vh;      // V*h
  u64 att_tok; // 2q + 2g
  u64 g2;      // 2g
  u64 kvb;     // 2*L*g*s
  u32 mml, pad;
};

// Per hardware profile: fp64 reciprocals (c.1) and the cost-model knobs.
struct DevHw {
  double invF, invB, invH, invT, overhead;
  u32 tp, pad;
};

// Per (hardware profile, policy) pair: block accounting (c.1).
struct DevHP {
  u64 total_blocks, block_bytes, ratio_limit, cap_fresh;
  u32 nwords, pad;
};

struct DevPol {
  u32 kind, preempt, mns, mbt, bs, wm;
  u32 bs_sh;  // log2(bs) if bs is a power of two, else 0xffffffff
  u32 mode;   // TOKENSIM_MIXED | TOKENSIM_PREFILL_FIRST | TOKENSIM_CHUNKED
};

// Per point, written once by the simulation kernel.
struct SimStats {
  u32 flags, pad;
  u64 n_finished, n_rejected, n_iterations, n_req_iters, n_preempt, swap_out, swap_in;
  i64 last_finish, t_final;
  u64 sched_d, block_d, req_d;
  u64 total_blocks, peak_blocks, block_ns_sum;
  u64 trace_n[8];  // per worker (x + y <= 8 for a P/D node); FULL: records in the stream
  u64 trace_b[8];  // FULL: bytes of each worker's compressed stream (trace_codec.cuh)
  u64 iter_n;
  u64 n_transfers, transfer_bytes;
  u64 ff_iters, ff_runs;  // iterations committed by fast-forward stretches, stretch count
  u64 cycles;             // SM clock cycles the warp spent on this point
  u64 cyc_ff, cyc_ff_fail, cyc_normal;  // cycles in stretches / failed attempts / normal iterations
  u64 phase[8];                         // stretch phases: pass/cost/list+alloc/update/fold/trace/compact/tail
  u64 nphase[8];                        // normal-iteration phases (see tokensim_point_profile)
  u64 n_req;                            // requests of this point (NEXT-2: rounds; else n_req)
  u64 ff_fail[5];                       // failed fast-forward attempts by reason (see the profile)
  u64 ff_cut[5];                        // what ended each stretch (see the profile)
};

// The model's cost-table coefficients as exact doubles (integers < 2^53), precomputed on the
// host so the kernels read them as constant-bank operands instead of holding them in registers.
struct DevModelF {
  double h, q2g, hq2g, qh, q, q4, hfu, fu, fh, f, Vh, V, s, att_tok, g2, L, twoL;
};
struct SweepParams {
  DevModel M;
  DevModelF MF;
  const DevHw *hw;      // [n_hw]
  const DevHP *hp;      // [n_hw * n_pol]
  const DevPol *pol;    // [n_pol]
  const double *rates;  // [n_rates]
  const u64 *seeds;     // [n_seeds]
  u32 n_hw, n_pol, n_rates, n_seeds;
  u32 topology, n_req;
  // workload: generated per (rate, seed) group; TRACE mode has one group
  u32 len_dist, n_groups;
  u32 prompt_a, prompt_b, output_a, output_b;
  const u32 *pt;  // prompt table: n | lo[n] | hi[n] | thr[n-1]   (device)
  const u32 *ot;  // output table
  const i64 *trace_a;
  const u32 *trace_p, *trace_o;
  i64 *arrival;   // [group][n]
  u32 *prompt;    // [group][n]
  u32 *output;    // [group][n]
  u32 group_of_point_mode;  // 0: (rate,seed) grid; 1: single TRACE group
  // run range (local index j -> point begin + j*stride)
  u64 begin, stride, n_run;
  const u32 *order;  // [n_run] local indices, longest-estimated first
  u32 *queue;        // [1] atomic work counter
  // outputs, indexed by local j
  tokensim_request_record *rec;  // [j][n]
  SimStats *stats;               // [j]
  tokensim_mem_sample *trace;    // [j][trace_nw][trace_cap]
  u32 trace_nw, bt_tables;       // workers per trace row (2, or x + y); block tables per warp
  u64 trace_cap;
  tokensim_iter_record *itrec;   // [j][it_cap]
  u64 it_cap;
  tokensim_summary *summ;        // [j]
  // per-warp scratch: block tables [warp][2][cap_slots][bt_len]
  u32 *bt;
  u32 bt_len, cap_slots, nwords_max, n_warps_total;
  u32 trace_mode, pad0;
  u64 bin_ns;
  i64 horizon, slo_ttft_ns, slo_mtpot_ns;
  double pd_link_inv;  // 1 / pd_link_bw
  u64 *scratch;        // summary keys when n_req exceeds the shared-memory key buffer
  u32 ff_enable, pad1; // time-parallel evaluation of quiescent decode stretches (H3)
  u32 *pd_ring;        // P/D: per-warp ring of P block ids [warp][pd_ring_len]
  u64 pd_ring_len;
  unsigned char *pd_fifo;  // P/D: per-warp pending/transfer FIFO [warp][n_req] x 32 B
  unsigned char *pdn_scratch;  // NEXT-1 node: per-CTA FIFOs, queues, holders, P block lists
  u64 pdn_bytes_per_warp;
  u32 pd_x, pd_y, dispatch, pd_general;  // prefill / decode workers, global scheduler, node loop
  u32 node_two, node_sw;   // node kernel: the register-capped two-CTAs-per-SM build; the scheduler-warp build
  u32 full, all_p2;                       // 1: the full kernel variant (sim_full.cu); every block size a power of two
  u32 n_sms, helper_mode;                 // SMs of the device; lean kernel with a helper warp per point: 1 = with
                                          // extended stretches (variant 0), 2 = without (variant 5)
  u32 n_heads, pad6;                      // variant 0: the first n_heads points (LPT order) each get an SM alone
  u32 *sched;                             // variant 0 with heads: per-SM arrival counts [256], SM states [256],
                                          // head ticket [1], head claims [n_heads] (zeroed per run)
  u32 link_mode, pad2;                    // NEXT-4: TOKENSIM_LINK_SEQUENTIAL | PRELOAD
  u64 preload_buf;                        // preload buffer bytes
  // NEXT-2 multi-round conversations + memory cache.  With multi_round, n_req = 7 * n_conv is
  // the per-group / per-point request stride and arrival/prompt/output are indexed by request
  // (rid = base[conv] + round; arrival holds round 0's arrival or round r's think gap).
  u32 multi_round, memory_cache, n_conv, pad3;
  double think_ns, fetch_s;
  u64 cache_cap;                          // blocks; 0 = 4 x the point's device KV blocks
  u32 *mr_conv;                           // [group][n_req] conversation of each request
  u32 *mr_base, *mr_nr;                   // [group][n_conv] first rid, number of rounds
  u32 *mr_ntot;                           // [group] requests
  i64 *mr_a0;                             // [group][n_conv] round-0 stream (a.1 output)
  u32 *mr_p0, *mr_o0;
  unsigned char *mr_scratch;              // per warp: arrival FIFO, follow-up heap, LRU cache
  u64 mr_bytes_per_warp;
  uint4 *evlog;            // per-warp block-event log [warp][1024]
  ulonglong2 *itlog;       // per-warp iteration log [warp][256][4]
  double *pipe;            // helper-warp full kernel: per-warp preload-pipeline scratch
  u64 pipe_stride;          // doubles per warp (>= layers + 1)
};

// point -> grid coordinates (row-major)
struct Coords {
  u32 hw, pol, rate, seed;
};
__host__ __device__ inline Coords decode_point(u64 point, u32 n_pol, u32 n_rates, u32 n_seeds) {
  Coords c;
  c.seed = (u32)(point % n_seeds);
  point /= n_seeds;
  c.rate = (u32)(point % n_rates);
  point /= n_rates;
  c.pol = (u32)(point % n_pol);
  c.hw = (u32)(point / n_pol);
  return c;
}

// launchers (sweep.cu)
cudaError_t launch_workload(const SweepParams &p, cudaStream_t st);
// kernel variants: 0 lean unified (helper warp + extended stretches), 1 full unified, 2 1P:1D pair,
// 3 xP:yD node (sim_node_kernel), 4 lean with compact helpers, 5 lean with the helper warp only,
// 6 full with the helper warp
cudaError_t launch_sim_base(const SweepParams &p, int cap, int warps_per_block, int blocks, size_t smem,
                            cudaStream_t st);
cudaError_t launch_sim_full(const SweepParams &p, int cap, int warps_per_block, int blocks, size_t smem,
                            cudaStream_t st);
cudaError_t launch_sim_full_h(const SweepParams &p, int cap, int warps_per_block, int blocks, size_t smem,
                              cudaStream_t st);
cudaError_t launch_sim_pair(const SweepParams &p, int cap, int warps_per_block, int blocks, size_t smem,
                            cudaStream_t st);
cudaError_t launch_sim_node(const SweepParams &p, int cap, int warps_per_block, int blocks, size_t smem,
                            cudaStream_t st);
cudaError_t launch_sim_base_c(const SweepParams &p, int cap, int warps_per_block, int blocks, size_t smem,
                              cudaStream_t st);
cudaError_t launch_sim_base_n(const SweepParams &p, int cap, int warps_per_block, int blocks, size_t smem,
                              cudaStream_t st);
// several warps per SM: the lean kernel with compact helpers (variant 4); one warp per SM:
// variant 0, whose CTA adds a helper warp (sim_base.cu)
// Shared memory of a variant-0 CTA: the simulating warp's area, then the helper's hand-over
// counters (kHelperChanBytes >= sizeof(HelperChan), asserted in sim_core.cuh), its replayed
// bitmap (nwords_max words) and 256 extraction slots.  A point whose CTA would not fit in
// 227 KB runs in variant 4 (no helper) instead.
constexpr size_t kHelperChanBytes = 128;
inline size_t helper_cta_smem(size_t per_warp, u32 nwords_max) {
  return ((per_warp + 15) & ~(size_t)15) + kHelperChanBytes + 4 * (size_t)nwords_max + 1024;
}
inline bool helper_fits(size_t per_warp, u32 nwords_max) { return helper_cta_smem(per_warp, nwords_max) <= 227 * 1024; }
// xs: the helper kernel with extended stretches (variant 0) rather than without (variant 5)
inline int sim_variant(bool full, bool pd, bool pd_general, bool multi_warp = false, bool xs = true) {
  return !full ? (multi_warp ? 4 : xs ? 0 : 5) : !pd ? (multi_warp ? 1 : 6) : pd_general ? 3 : 2;
}
inline cudaError_t launch_sim(const SweepParams &p, int cap, int warps_per_block, int blocks, size_t smem,
                              cudaStream_t st) {
  (void)blocks;
  switch (sim_variant(p.full != 0, p.topology == TOKENSIM_PD_PAIR, p.pd_general != 0,
                      !(p.helper_mode && warps_per_block == 1 && helper_fits(smem, p.nwords_max)), p.helper_mode == 1)) {
    case 0: return launch_sim_base(p, cap, warps_per_block, blocks, smem, st);
    case 5: return launch_sim_base_n(p, cap, warps_per_block, blocks, smem, st);
    case 4: return launch_sim_base_c(p, cap, warps_per_block, blocks, smem, st);
    case 1: return launch_sim_full(p, cap, warps_per_block, blocks, smem, st);
    case 6: return launch_sim_full_h(p, cap, warps_per_block, blocks, smem, st);
    case 2: return launch_sim_pair(p, cap, warps_per_block, blocks, smem, st);
    default: return launch_sim_node(p, cap, warps_per_block, blocks, smem, st);
  }
}
cudaError_t launch_summary(const SweepParams &p, cudaStream_t st);
cudaError_t launch_quantiles(const SweepParams &p, u64 j, u32 metric, const u32 *d_ranks, u32 n_q,
                             double *d_out, u64 *d_keys, cudaStream_t st);
constexpr u32 kSummarySmemKeys = 12288;  // keys held in shared memory by summary_kernel
size_t sim_smem_per_warp(int cap, u32 nwords_max, bool pd, u32 node_x, u32 node_y);
// NEXT-1 node, global scratch per CTA (one point): decode FIFOs [y][n] x 32 B, prefill queues and holder
// lists [x][n] x 4 B each, in-flight batches [x][cap] x 4 B, transfer ends [n] x 8 B, prefill
// block lists [n][bt_len] x 4 B (sim_pdn.cuh)
inline size_t pdn_global_per_warp(u64 n, u32 cap, u32 btl, u32 x, u32 y) {
  return (size_t)y * n * 32 + (size_t)x * n * 4 * 2 + (size_t)x * cap * 4 + n * 8 + n * (size_t)btl * 4 + 256;
}
cudaError_t sim_occupancy_base(int cap, int warps_per_block, size_t smem, u32 nwords_max, int *blocks_per_sm);
cudaError_t sim_occupancy_full(int cap, int warps_per_block, size_t smem, u32 nwords_max, int *blocks_per_sm);
cudaError_t sim_occupancy_full_h(int cap, int warps_per_block, size_t smem, u32 nwords_max, int *blocks_per_sm);
cudaError_t sim_occupancy_pair(int cap, int warps_per_block, size_t smem, u32 nwords_max, int *blocks_per_sm);
// (node: warps_per_block = the CTA's warps, + 16 for the two-CTAs-per-SM build, + 32 for the scheduler-warp build)
cudaError_t sim_occupancy_node(int cap, int warps_per_block, size_t smem, u32 nwords_max, int *blocks_per_sm);
cudaError_t sim_occupancy_base_c(int cap, int warps_per_block, size_t smem, u32 nwords_max, int *blocks_per_sm);
cudaError_t sim_occupancy_base_n(int cap, int warps_per_block, size_t smem, u32 nwords_max, int *blocks_per_sm);
inline cudaError_t sim_occupancy(int variant, int cap, int warps_per_block, size_t smem, u32 nwords_max,
                                 int *blocks_per_sm) {
  switch (variant) {
    case 0: return sim_occupancy_base(cap, warps_per_block, smem, nwords_max, blocks_per_sm);
    case 1: return sim_occupancy_full(cap, warps_per_block, smem, nwords_max, blocks_per_sm);
    case 6: return sim_occupancy_full_h(cap, warps_per_block, smem, nwords_max, blocks_per_sm);
    case 2: return sim_occupancy_pair(cap, warps_per_block, smem, nwords_max, blocks_per_sm);
    case 4: return sim_occupancy_base_c(cap, warps_per_block, smem, nwords_max, blocks_per_sm);
    case 5: return sim_occupancy_base_n(cap, warps_per_block, smem, nwords_max, blocks_per_sm);
    default: return sim_occupancy_node(cap, warps_per_block, smem, nwords_max, blocks_per_sm);
  }
}

}  // namespace ts
