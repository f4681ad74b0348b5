// host.cu -- the C ABI (include/tokensim.h): validation, derived constants (SURVEY c.1),
// device tables, workspace layout, launch sequence and result getters.
//
// The host only marshals: every step of the sweep (a.1-a.8) runs in the kernels of
// sweep.cu.  Derived per-profile constants are computed here once per create (they are
// inputs of the simulation, like the profile itself), in the fp64 order of SURVEY c.1.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only: ranges cost nothing unless a profiler injects itself

#include "ts_internal.cuh"

using namespace ts;

namespace {

thread_local std::string g_create_err;

// SHAREGPT_SYNTH_V1 (reading A25): bucket bounds and u32 thresholds.
const uint32_t kPromptLo[7] = {4, 16, 32, 64, 128, 256, 512};
const uint32_t kPromptHi[7] = {16, 32, 64, 128, 256, 512, 1024};
const uint32_t kPromptThr[6] = {644245094u, 1309965025u, 2040109466u, 2770253906u, 3457448673u, 3994319585u};
const uint32_t kOutputLo[8] = {4, 16, 32, 64, 128, 256, 512, 1024};
const uint32_t kOutputHi[8] = {16, 32, 64, 128, 256, 512, 1024, 2048};
const uint32_t kOutputThr[7] = {429496730u, 773094113u, 1159641170u, 1717986918u, 2448131359u, 3307124818u,
                                4101693768u};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
  size_t arrival, prompt, output, rec, stats, trace, itrec, summ, bt, order, queue, sched, scratch, ring, fifo, pdn,
      pdn_per_warp,
      mr_conv, mr_base, mr_nr, mr_ntot, mr_a0, mr_p0, mr_o0, mr, mr_per_warp, evlog, itlog, pipe, pipe_stride,
      total;
  u64 n_run;
  u32 warps_total, wpb, blocks;
  size_t smem;
};

}  // namespace

struct tokensim_sweep {
  tokensim_model model{};
  std::vector<tokensim_hw> hw;
  std::vector<tokensim_policy> pol;
  std::vector<double> rates;
  std::vector<uint64_t> seeds;
  tokensim_workload wl{};
  tokensim_options opt{};
  std::vector<uint32_t> ptab, otab;  // n | lo | hi | thr
  std::vector<int64_t> tr_a;
  std::vector<uint32_t> tr_p, tr_o;
  // derived
  DevModel M{};
  std::vector<DevHw> dhw;
  std::vector<DevHP> dhp;
  std::vector<DevPol> dpol;
  std::vector<double> est_T1;  // per (hw,pol): rough per-iteration time for LPT ordering
  // per (hw,pol) inputs of the LPT cost estimate (lpt_cost): weights / bandwidth, KV read time
  // per context token, decode FLOP time per token, the overhead, and the memory-bound batch
  struct EstHP {
    double w_s, tok_s, flop_s, ovh, bmem, bmax;
    bool stat;  // static batching
  };
  std::vector<EstHP> est_hp;
  double mean_p = 0, mean_o = 0;  // workload means (table / fixed / uniform / trace)
  u32 cap = 256, nwords_max = 1, bt_len = 1, n_hw_axis = 0;
  u32 pd_x = 0, pd_y = 0;  // NEXT-1 node: prefill / decode workers (0 = unified)
  bool pd_general = false;  // run the general xP:yD loop
  bool full = false;        // needs the full kernel variant (sim_full.cu)
  u32 trace_nw() const { return pd_general ? std::max<u32>(2, pd_x + pd_y) : 2; }
  u32 bt_tables() const { return pd_general ? pd_y + 1 : 2; }
  // requests per point (record stride): 7 x conversations with multi-round workloads
  u64 n_slots() const { return wl.multi_round ? 7ull * wl.num_requests : (u64)wl.num_requests; }
  size_t smem_per_warp() const {
    return sim_smem_per_warp((int)cap, nwords_max, opt.topology == TOKENSIM_PD_PAIR, pd_general ? pd_x : 0,
                             pd_general ? pd_y : 0);
  }
  u64 n_points = 0, max_total_blocks = 0;
  // device tables
  int dev = -1;
  char *d_tab = nullptr;
  size_t off_hw = 0, off_hp = 0, off_pol = 0, off_rates = 0, off_seeds = 0, off_pt = 0, off_ot = 0,
         off_tra = 0, off_trp = 0, off_tro = 0;
  // last run
  bool ran = false;
  u64 begin = 0, end = 0, stride = 1, n_run = 0;
  char *ws = nullptr;
  size_t ws_bytes = 0;
  char *owned_ws = nullptr;
  size_t owned_bytes = 0;
  cudaStream_t stream = nullptr;
  SweepParams P{};
  Layout lay{};
  std::vector<tokensim_summary> imported;  // indexed by point; version 0 = absent
  std::string err;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  u32 n_launches = 0;
  u64 h2d_bytes = 0, table_bytes_pending = 0;
};

namespace {

tokensim_status fail(tokensim_sweep *h, tokensim_status s, const std::string &m) {
  if (h) h->err = m;
  else g_create_err = m;
  return s;
}
tokensim_status cuda_fail(tokensim_sweep *h, cudaError_t e, const char *what) {
  return fail(h, TOKENSIM_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }

// ---- c.1 derived constants (host side of the product; independent of oracle/)
u64 weight_bytes(const tokensim_model &m) {
  const u64 L = m.num_layers, h = m.hidden, V = m.vocab, f = m.ffn_dim, s = m.dtype_bytes;
  const u64 q = (u64)m.num_heads * m.head_dim, g = (u64)m.num_kv_heads * m.head_dim;
  const u64 layer = h * (q + 2 * g) + q * h + (m.gated_mlp ? 3 : 2) * h * f;
  return s * (L * layer + (m.tied_embeddings ? 1 : 2) * V * h + (2 * L + 1) * h);
}

std::string hwpath(u32 i, const char *f) { return "hw[" + std::to_string(i) + "]." + f; }

}  // namespace

extern "C" {

const char *tokensim_version(void) { return "tokensim-b200 1 sm_100a"; }

const char *tokensim_last_error(const tokensim_sweep *h) {
  return h ? h->err.c_str() : g_create_err.c_str();
}

tokensim_status tokensim_sweep_create(const tokensim_model *model, const tokensim_hw *hw, uint32_t n_hw,
                                      const tokensim_policy *pol, uint32_t n_pol,
                                      const tokensim_workload *wl, const tokensim_options *opt,
                                      tokensim_sweep **out) {
  g_create_err.clear();
  if (!out) return fail(nullptr, TOKENSIM_E_INVALID, "out: NULL");
  *out = nullptr;
  if (!model || !hw || !pol || !wl || !opt) return fail(nullptr, TOKENSIM_E_INVALID, "NULL input struct");
  if (model->struct_size != sizeof(tokensim_model)) return fail(nullptr, TOKENSIM_E_INVALID, "model.struct_size mismatch");
  if (wl->struct_size != sizeof(tokensim_workload)) return fail(nullptr, TOKENSIM_E_INVALID, "workload.struct_size mismatch");
  if (opt->struct_size != sizeof(tokensim_options)) return fail(nullptr, TOKENSIM_E_INVALID, "options.struct_size mismatch");
  if (n_hw == 0) return fail(nullptr, TOKENSIM_E_INVALID, "n_hw: must be >= 1");
  if (n_pol == 0) return fail(nullptr, TOKENSIM_E_INVALID, "n_pol: must be >= 1");
  for (u32 i = 0; i < n_hw; ++i)
    if (hw[i].struct_size != sizeof(tokensim_hw)) return fail(nullptr, TOKENSIM_E_INVALID, hwpath(i, "struct_size") + " mismatch");
  for (u32 i = 0; i < n_pol; ++i)
    if (pol[i].struct_size != sizeof(tokensim_policy))
      return fail(nullptr, TOKENSIM_E_INVALID, "policies[" + std::to_string(i) + "].struct_size mismatch");

  const tokensim_model &m = *model;
  if (!m.num_layers || !m.hidden || !m.num_heads || !m.num_kv_heads || !m.head_dim || !m.ffn_dim || !m.vocab ||
      !m.dtype_bytes)
    return fail(nullptr, TOKENSIM_E_INVALID, "model: every dimension must be >= 1");
  if (m.max_model_len < 2 || m.max_model_len > (1u << 20))
    return fail(nullptr, TOKENSIM_E_INVALID, "model.max_model_len: must be in [2, 2^20]");
  if (opt->topology > TOKENSIM_PD_PAIR) return fail(nullptr, TOKENSIM_E_INVALID, "options.topology: unknown");
  if (opt->topology == TOKENSIM_PD_PAIR && !(opt->pd_link_bw > 0))
    return fail(nullptr, TOKENSIM_E_INVALID, "options.pd_link_bw: must be > 0 with PD_PAIR");
  if (opt->link_mode > TOKENSIM_LINK_PRELOAD) return fail(nullptr, TOKENSIM_E_INVALID, "options.link_mode: unknown");
  if (opt->link_mode == TOKENSIM_LINK_PRELOAD && opt->preload_buffer_bytes == 0)
    return fail(nullptr, TOKENSIM_E_INVALID, "options.preload_buffer_bytes: must be > 0 with PRELOAD");
  if (opt->link_mode == TOKENSIM_LINK_PRELOAD && m.num_layers > 2000)
    return fail(nullptr, TOKENSIM_E_INVALID, "model.num_layers: at most 2000 with a PRELOAD link");
  if (opt->topology == TOKENSIM_PD_PAIR) {
    const u32 x = opt->pd_prefill_workers ? opt->pd_prefill_workers : 1u;
    const u32 y = opt->pd_decode_workers ? opt->pd_decode_workers : 1u;
    if (x + y > 8) return fail(nullptr, TOKENSIM_E_INVALID, "options.pd_prefill_workers + pd_decode_workers: at most 8");
    if (opt->dispatch > TOKENSIM_DISPATCH_LEAST_MEMORY)
      return fail(nullptr, TOKENSIM_E_INVALID, "options.dispatch: unknown");
  }
  if (opt->trace_mode > TOKENSIM_TRACE_FULL) return fail(nullptr, TOKENSIM_E_INVALID, "options.trace_mode: unknown");
  if (opt->trace_mode == TOKENSIM_TRACE_BINNED && opt->trace_bin_ns == 0)
    return fail(nullptr, TOKENSIM_E_INVALID, "options.trace_bin_ns: must be > 0");
  if (!(opt->slo_ttft_s >= 0) || !(opt->slo_mtpot_s >= 0))
    return fail(nullptr, TOKENSIM_E_INVALID, "options.slo_*: must be >= 0");

  const tokensim_workload &w = *wl;
  if (w.num_requests == 0) return fail(nullptr, TOKENSIM_E_INVALID, "workload.num_requests: must be >= 1");
  if (w.num_requests > (1u << 30)) return fail(nullptr, TOKENSIM_E_INVALID, "workload.num_requests: too large");
  if (w.num_rates == 0 || !w.rates) return fail(nullptr, TOKENSIM_E_INVALID, "workload.rates: empty");
  if (w.num_seeds == 0 || !w.seeds) return fail(nullptr, TOKENSIM_E_INVALID, "workload.seeds: empty");
  for (u32 i = 0; i < w.num_rates; ++i)
    if (!(w.rates[i] > 0) || !std::isfinite(w.rates[i]))
      return fail(nullptr, TOKENSIM_E_INVALID, "workload.rates[" + std::to_string(i) + "]: must be > 0");

  tokensim_sweep *h = new tokensim_sweep();
  h->model = m;
  h->hw.assign(hw, hw + n_hw);
  h->pol.assign(pol, pol + n_pol);
  h->rates.assign(w.rates, w.rates + w.num_rates);
  h->seeds.assign(w.seeds, w.seeds + w.num_seeds);
  h->wl = w;
  h->opt = *opt;
  const u32 mml = m.max_model_len;
  auto bad = [&](const std::string &msg) {
    delete h;
    return fail(nullptr, TOKENSIM_E_INVALID, msg);
  };

  // ---- workload lengths
  auto load_table = [&](const tokensim_len_table *t, const char *name, std::vector<u32> &dst, u32 max_hi,
                        std::string &e) -> bool {
    if (!t || t->n_buckets == 0 || !t->lo || !t->hi || (t->n_buckets > 1 && !t->cdf32)) {
      e = std::string("workload.") + name + ": missing table";
      return false;
    }
    dst.clear();
    dst.push_back(t->n_buckets);
    for (u32 b = 0; b < t->n_buckets; ++b) {
      if (t->lo[b] < 1 || t->hi[b] <= t->lo[b] || t->hi[b] > max_hi + 1) {
        e = std::string("workload.") + name + ".bucket[" + std::to_string(b) + "]: need 1 <= lo < hi <= " +
            std::to_string(max_hi + 1);
        return false;
      }
    }
    for (u32 b = 0; b < t->n_buckets; ++b) dst.push_back(t->lo[b]);
    for (u32 b = 0; b < t->n_buckets; ++b) dst.push_back(t->hi[b]);
    for (u32 b = 0; b + 1 < t->n_buckets; ++b) {
      if (b && t->cdf32[b] < t->cdf32[b - 1]) {
        e = std::string("workload.") + name + ".cdf32: must be non-decreasing";
        return false;
      }
      dst.push_back(t->cdf32[b]);
    }
    dst.push_back(0);
    return true;
  };
  std::string e;
  switch (w.len_dist) {
    case TOKENSIM_LEN_SHAREGPT_SYNTH_V1: {
      if (mml < 2048) return bad("workload.len_dist: SHAREGPT_SYNTH_V1 needs max_model_len >= 2048");
      tokensim_len_table pt = {7, kPromptLo, kPromptHi, kPromptThr}, ot = {8, kOutputLo, kOutputHi, kOutputThr};
      load_table(&pt, "prompt_table", h->ptab, mml - 1, e);
      load_table(&ot, "output_table", h->otab, 1u << 30, e);
      break;
    }
    case TOKENSIM_LEN_TABLE:
      if (!load_table(w.prompt_table, "prompt_table", h->ptab, mml - 1, e)) return bad(e);
      if (!load_table(w.output_table, "output_table", h->otab, 1u << 30, e)) return bad(e);
      break;
    case TOKENSIM_LEN_FIXED:
      if (w.prompt_a < 1 || w.output_a < 1 || (u64)w.prompt_a + w.output_a > mml)
        return bad("workload.prompt_a/output_a: need >= 1 and prompt + output <= max_model_len");
      break;
    case TOKENSIM_LEN_UNIFORM:
      if (w.prompt_a < 1 || w.prompt_b < w.prompt_a || w.prompt_b > mml - 1 || w.output_a < 1 ||
          w.output_b < w.output_a)
        return bad("workload.prompt_[ab]/output_[ab]: need 1 <= a <= b, prompt_b < max_model_len");
      break;
    case TOKENSIM_LEN_TRACE: {
      if (w.num_rates != 1 || w.num_seeds != 1)
        return bad("workload: TRACE mode takes exactly one rate and one seed (they are unused)");
      if (!w.trace_arrival_ns || !w.trace_prompt || !w.trace_output) return bad("workload.trace_*: NULL");
      h->tr_a.assign(w.trace_arrival_ns, w.trace_arrival_ns + w.num_requests);
      h->tr_p.assign(w.trace_prompt, w.trace_prompt + w.num_requests);
      h->tr_o.assign(w.trace_output, w.trace_output + w.num_requests);
      for (u32 i = 0; i < w.num_requests; ++i) {
        if (h->tr_a[i] < 0 || (i && h->tr_a[i] < h->tr_a[i - 1]))
          return bad("workload.trace_arrival_ns[" + std::to_string(i) + "]: must be >= 0 and non-decreasing");
        if (h->tr_p[i] < 1 || h->tr_o[i] < 1 || (u64)h->tr_p[i] + h->tr_o[i] > mml)
          return bad("workload.trace[" + std::to_string(i) + "]: need prompt, output >= 1 and sum <= max_model_len");
      }
      break;
    }
    default:
      return bad("workload.len_dist: unknown");
  }
  // NEXT-2 multi-round conversations and the memory cache (reading R-N2)
  if (w.multi_round) {
    if (w.len_dist == TOKENSIM_LEN_TRACE) return bad("workload.multi_round: needs generated lengths, not TRACE");
    if (opt->topology != TOKENSIM_UNIFIED) return bad("workload.multi_round: UNIFIED topology only");
    if (!(w.think_mean_s >= 0) || !std::isfinite(w.think_mean_s)) return bad("workload.think_mean_s: must be >= 0");
    if ((u64)w.num_requests * 7 > (1u << 30)) return bad("workload.num_requests: too many conversations");
    for (u32 i = 0; i < n_pol; ++i)
      if (pol[i].iteration_mode != TOKENSIM_MIXED) return bad("workload.multi_round: MIXED iterations only");
  }
  if (opt->memory_cache && !w.multi_round) return bad("options.memory_cache: needs a multi_round workload");
  {  // workload length means, for the LPT cost estimate only (lpt_cost)
    auto tab_mean = [](const std::vector<u32> &t) {
      const u32 nb = t[0];
      const u32 *lo = &t[1], *hi = &t[1 + nb], *thr = &t[1 + 2 * nb];
      double prev = 0, m = 0;
      for (u32 b = 0; b < nb; ++b) {
        const double c = b + 1 < nb ? (double)thr[b] : 4294967296.0;
        m += (c - prev) / 4294967296.0 * ((double)lo[b] + ((double)hi[b] - lo[b] - 1) / 2.0);
        prev = c;
      }
      return m;
    };
    if (!h->ptab.empty() && !h->otab.empty()) {
      h->mean_p = tab_mean(h->ptab);
      h->mean_o = std::min(tab_mean(h->otab), (double)mml - h->mean_p);
    } else if (w.len_dist == TOKENSIM_LEN_FIXED) {
      h->mean_p = w.prompt_a;
      h->mean_o = w.output_a;
    } else if (w.len_dist == TOKENSIM_LEN_UNIFORM) {
      h->mean_p = 0.5 * ((double)w.prompt_a + w.prompt_b);
      h->mean_o = 0.5 * ((double)w.output_a + w.output_b);
    } else {
      double sp = 0, so = 0;
      for (u32 i = 0; i < w.num_requests; ++i) {
        sp += h->tr_p[i];
        so += h->tr_o[i];
      }
      h->mean_p = sp / std::max<u32>(1, w.num_requests);
      h->mean_o = so / std::max<u32>(1, w.num_requests);
    }
  }
  if (!(opt->cache_fetch_ns_per_block >= 0) || !std::isfinite(opt->cache_fetch_ns_per_block))
    return bad("options.cache_fetch_ns_per_block: must be >= 0");

  // ---- model constants
  DevModel &M = h->M;
  M.L = m.num_layers;
  M.h = m.hidden;
  M.q = (u64)m.num_heads * m.head_dim;
  M.g = (u64)m.num_kv_heads * m.head_dim;
  M.f = m.ffn_dim;
  M.fu = m.gated_mlp ? 2 * (u64)m.ffn_dim : (u64)m.ffn_dim;
  M.V = m.vocab;
  M.s = m.dtype_bytes;
  M.q2g = M.q + 2 * M.g;
  M.hq2g = M.h * M.q2g;
  M.qh = M.q * M.h;
  M.hfu = M.h * M.fu;
  M.fh = M.f * M.h;
  M.Vh = M.V * M.h;
  M.att_tok = 2 * M.q + 2 * M.g;
  M.g2 = 2 * M.g;
  M.kvb = 2 * M.L * M.g * M.s;
  M.mml = mml;
  const u64 W = weight_bytes(m);

  // ---- policies
  u32 max_mns = 1, min_bs = 0xffffffffu;
  bool any_swap = false;
  for (u32 i = 0; i < n_pol; ++i) {
    const tokensim_policy &p = pol[i];
    const std::string pp = "policies[" + std::to_string(i) + "].";
    if (p.kind > TOKENSIM_CONT_RATIO) return bad(pp + "kind: unknown");
    if (p.preempt > TOKENSIM_RECOMPUTE) return bad(pp + "preempt: unknown");
    if (p.iteration_mode > TOKENSIM_CHUNKED) return bad(pp + "iteration_mode: unknown");
    if (opt->topology == TOKENSIM_PD_PAIR && p.iteration_mode != TOKENSIM_MIXED)
      return bad(pp + "iteration_mode: PD_PAIR workers are prefill-only / decode-only already");
    if (opt->topology == TOKENSIM_PD_PAIR && p.kind == TOKENSIM_CONT_RATIO)
      return bad(pp + "kind: PD_PAIR supports STATIC and CONT (reading R-PD1)");
    if (p.kind == TOKENSIM_CONT_RATIO && !(p.max_mem_ratio > 0 && p.max_mem_ratio <= 1))
      return bad(pp + "max_mem_ratio: must be in (0, 1]");
    if (p.max_num_seqs < 1 || p.max_num_seqs > 1024) return bad(pp + "max_num_seqs: must be in [1, 1024]");
    if (p.iteration_mode == TOKENSIM_CHUNKED) {
      // every running decode must fit the budget (reading R-N3b); prompts are chunked
      if (p.max_batched_tokens < p.max_num_seqs)
        return bad(pp + "max_batched_tokens: CHUNKED needs max_batched_tokens >= max_num_seqs");
    } else if (p.max_batched_tokens < mml) {
      return bad(pp + "max_batched_tokens: must be >= max_model_len");
    }
    if (p.block_size < 1) return bad(pp + "block_size: must be >= 1");
    max_mns = std::max(max_mns, p.max_num_seqs);
    min_bs = std::min(min_bs, p.block_size);
    any_swap |= p.preempt == TOKENSIM_SWAP;
    DevPol d;
    d.kind = p.kind;
    d.preempt = p.preempt;
    d.mns = p.max_num_seqs;
    d.mbt = p.max_batched_tokens;
    d.bs = p.block_size;
    d.wm = p.watermark_blocks;
    d.bs_sh = (p.block_size & (p.block_size - 1)) ? 0xffffffffu : (u32)__builtin_ctz(p.block_size);
    d.mode = p.iteration_mode;
    h->dpol.push_back(d);
  }
  h->cap = max_mns <= 32 ? 32 : (max_mns <= 256 ? 256 : 1024);
  h->bt_len = (u32)ceil_div(mml, min_bs);
  if (h->bt_len > (1u << 17)) return bad("model.max_model_len / policies[].block_size: more than 2^17 blocks per request");
  // every F_o / B_o of the c.5 cost table must stay an exact fp64 integer (< 2^53)
  {
    typedef unsigned __int128 u128;
    const u128 lim = (u128)1 << 53;
    u128 worst = 0;
    for (u32 i = 0; i < n_pol; ++i) {
      const u128 mns = pol[i].max_num_seqs;
      const u128 Np = std::min<u128>(pol[i].max_batched_tokens, mns * mml);
      const u128 N = Np + mns, S = mns;
      const u128 Ap = mns * (u128)mml * (mml + 1) / 2, Cd = mns * (u128)(mml + 1);
      // chunks (CHUNKED): A_p <= N_p * mml and K_p <= N_p + mns * mml
      const bool chk = pol[i].iteration_mode == TOKENSIM_CHUNKED;
      const u128 Apc = chk ? Np * (u128)mml : 0, Kpc = chk ? Np + mns * (u128)mml : Np;
      const u128 Ab = Ap > Apc ? Ap : Apc, Kb = Kpc > Cd ? Kpc : Cd;
      const u128 cand[] = {2 * N * M.hq2g, M.s * (M.hq2g + N * M.h + N * M.q2g), 2 * N * M.hfu,
                           M.s * (M.hfu + N * M.h + N * M.fu), 4 * (u128)M.q * Ab, 4 * (u128)M.q * Cd,
                           M.s * (N * M.att_tok + M.g2 * Kb), 2 * S * M.Vh,
                           M.s * (M.Vh + S * M.h + S * M.V)};
      for (u128 c : cand) worst = std::max(worst, c);
    }
    if (worst >= lim) return bad("model x policies: cost-table integers exceed 2^53 (not exact in fp64)");
  }

  // ---- hardware profiles and (hw, pol) block accounting
  u64 max_words = 1;
  for (u32 i = 0; i < n_hw; ++i) {
    const tokensim_hw &x = hw[i];
    if (!(x.peak_flops > 0) || !(x.mem_bw > 0) || !std::isfinite(x.peak_flops) || !std::isfinite(x.mem_bw))
      return bad(hwpath(i, "peak_flops/mem_bw") + ": must be finite and > 0");
    if (!(x.eff_flops > 0 && x.eff_flops <= 1) || !(x.eff_bw > 0 && x.eff_bw <= 1))
      return bad(hwpath(i, "eff_flops/eff_bw") + ": must be in (0, 1]");
    if (!(x.reserve_frac >= 0 && x.reserve_frac < 1)) return bad(hwpath(i, "reserve_frac") + ": must be in [0, 1)");
    if (!(x.iter_overhead_s >= 0)) return bad(hwpath(i, "iter_overhead_s") + ": must be >= 0");
    if (x.tp_degree < 1) return bad(hwpath(i, "tp_degree") + ": must be >= 1");
    if (x.tp_degree > 1 && !(x.tp_link_bw > 0)) return bad(hwpath(i, "tp_link_bw") + ": must be > 0 when tp_degree > 1");
    if (any_swap && !(x.host_link_bw > 0)) return bad(hwpath(i, "host_link_bw") + ": must be > 0 with SWAP");
    DevHw d;
    d.invF = 1.0 / (x.peak_flops * x.eff_flops);
    d.invB = 1.0 / (x.mem_bw * x.eff_bw);
    d.invH = x.host_link_bw > 0 ? 1.0 / x.host_link_bw : 0.0;
    d.invT = x.tp_degree > 1 ? 1.0 / ((double)x.tp_degree * x.tp_link_bw) : 0.0;
    d.overhead = x.iter_overhead_s;
    d.tp = x.tp_degree;
    d.pad = 0;
    h->dhw.push_back(d);
    const u64 reserve = (u64)std::floor((double)x.mem_capacity * x.reserve_frac);
    for (u32 j = 0; j < n_pol; ++j) {
      const tokensim_policy &p = pol[j];
      DevHP hp;
      hp.block_bytes = (u64)p.block_size * M.kvb;
      if (x.kv_blocks_override) {
        hp.total_blocks = x.kv_blocks_override;
      } else {
        if (x.mem_capacity < W + reserve)
          return bad(hwpath(i, "mem_capacity") + ": " + std::to_string(x.mem_capacity) + " < weights " +
                     std::to_string(W) + " + reserve " + std::to_string(reserve));
        hp.total_blocks = (x.mem_capacity - W - reserve) / hp.block_bytes;
      }
      const u64 min_blocks = ceil_div(mml, p.block_size);
      if (hp.total_blocks < min_blocks)
        return bad(hwpath(i, "mem_capacity") + ": " + std::to_string(hp.total_blocks) + " KV blocks of " +
                   std::to_string(p.block_size) + " tokens cannot hold one max_model_len request (policies[" +
                   std::to_string(j) + "])");
      if (hp.total_blocks > (1ull << 21))
        return bad(hwpath(i, "mem_capacity") + ": more than 2^21 KV blocks per worker is not supported");
      if ((u64)p.watermark_blocks > hp.total_blocks - min_blocks)
        return bad("policies[" + std::to_string(j) + "].watermark_blocks: must be <= total_blocks - ceil(max_model_len/block_size) = " +
                   std::to_string(hp.total_blocks - min_blocks) + " on hw[" + std::to_string(i) + "]");
      hp.ratio_limit = (u64)std::floor(p.max_mem_ratio * (double)hp.total_blocks);
      hp.cap_fresh = p.kind == TOKENSIM_CONT_RATIO ? hp.ratio_limit : hp.total_blocks - p.watermark_blocks;
      hp.nwords = (u32)ceil_div(hp.total_blocks, 32);
      hp.pad = 0;
      max_words = std::max<u64>(max_words, hp.nwords);
      h->dhp.push_back(hp);
      // LPT estimate: weights over bandwidth + overhead is the decode step floor
      h->est_T1.push_back((double)W / (x.mem_bw * x.eff_bw) + x.iter_overhead_s);
      {
        tokensim_sweep::EstHP e;
        const double Bw = x.mem_bw * x.eff_bw, Ff = x.peak_flops * x.eff_flops;  // aggregate profile (A22)
        e.w_s = (double)W / Bw;
        e.tok_s = (double)M.kvb / Bw;
        e.flop_s = (double)W / ((double)M.s * 0.5 * Ff);  // ~2 FLOPs per parameter per token
        e.ovh = x.iter_overhead_s;
        e.bmem = (double)hp.total_blocks * p.block_size;  // KV tokens (divided by the mean context later)
        if (p.kind == TOKENSIM_CONT_RATIO) e.bmem *= p.max_mem_ratio;
        e.bmax = p.max_num_seqs;
        e.stat = p.kind == TOKENSIM_STATIC;
        h->est_hp.push_back(e);
      }
    }
  }
  h->nwords_max = (u32)((max_words + 31) & ~31ull);
  h->n_hw_axis = n_hw;
  const u64 hw_axis = opt->topology == TOKENSIM_PD_PAIR ? (u64)n_hw * n_hw : (u64)n_hw;
  h->n_points = hw_axis * n_pol * w.num_rates * w.num_seeds;
  u64 max_total = 0;
  for (const DevHP &x : h->dhp) max_total = std::max(max_total, x.total_blocks);
  h->max_total_blocks = max_total;
  if (opt->topology == TOKENSIM_PD_PAIR) {
    h->pd_x = opt->pd_prefill_workers ? opt->pd_prefill_workers : 1u;
    h->pd_y = opt->pd_decode_workers ? opt->pd_decode_workers : 1u;
    h->pd_general = h->pd_x > 1 || h->pd_y > 1 || (opt->flags & TOKENSIM_OPT_NODE_LOOP);
  }
  h->full = opt->topology == TOKENSIM_PD_PAIR || w.multi_round || opt->memory_cache ||
            opt->link_mode == TOKENSIM_LINK_PRELOAD;
  // prefill-first and chunked iterations run in the full variant (the lean one keeps MIXED only)
  for (u32 i = 0; i < n_pol; ++i) h->full |= pol[i].iteration_mode != TOKENSIM_MIXED;
  const size_t per_warp = h->smem_per_warp();
  if (per_warp > 227 * 1024) {
    delete h;
    return fail(nullptr, TOKENSIM_E_INVALID, "max_num_seqs x total_blocks needs more than 227 KB of shared memory per point");
  }
  *out = h;
  return TOKENSIM_OK;
}

uint64_t tokensim_sweep_num_points(const tokensim_sweep *h) { return h ? h->n_points : 0; }
uint64_t tokensim_sweep_num_run(const tokensim_sweep *h) { return h && h->ran ? h->n_run : 0; }

static bool range_ok(const tokensim_sweep *h, u64 begin, u64 end, u64 stride) {
  return stride >= 1 && begin <= end && end <= h->n_points;
}
static u64 count_run(u64 begin, u64 end, u64 stride) { return end > begin ? (end - begin + stride - 1) / stride : 0; }

// LPT cost estimate of one unified-topology point (longest-estimated points start first).  A
// queueing sketch of the simulated system: decode step time T(b) = overhead + max(weights + b x
// context KV, b x decode FLOPs) at batch b; the batch the load sustains (Little's law on tokens,
// b = lambda E[o] T(b), capped by max_num_seqs and by the KV pool over the mean context);
// iterations = span / T(b) (or E[o] n / b_max when overloaded).  Simulation cost ~ 256 SM cycles
// per iteration, ~22k per admission iteration (one per request; static batching: one per batch)
// and ~14k more per request when the KV pool binds (preemption churn).  Fitted to round-2
// per-point cycle counts of C3; it only orders the queue, never changes a result.
static double lpt_cost(const tokensim_sweep *h, u32 hwpol, double rate, double *quiet = nullptr,
                       double *iters_out = nullptr) {
  const auto &e = h->est_hp[hwpol];
  const double n = h->wl.num_requests, Eo = std::max(1.0, h->mean_o), ctx = h->mean_p + 0.5 * Eo;
  const double bmem = std::max(1.0, e.bmem / std::max(1.0, ctx));
  const double bmax = std::max(1.0, std::min(e.bmax, bmem));
  auto T = [&](double b) { return e.ovh + std::max(e.w_s + b * ctx * e.tok_s, b * e.flop_s); };
  double b = bmax, iters;
  if (rate * Eo >= bmax / T(bmax)) {
    iters = n * Eo / bmax;
  } else {
    b = 1.0;
    for (int it = 0; it < 30; ++it) b = std::min(bmax, std::max(1.0, rate * Eo * T(b)));
    iters = (n / rate) / T(b);
  }
  // churn: Poisson arrivals and the length spread fill a memory-limited pool well before the
  // mean batch reaches it (C4 TP2 at lambda 4: b ~ 0.46 b_max, ~1.3 preemptions per request)
  // iterations between two events (an arrival or a finish, each at rate lambda in steady state)
  if (quiet) *quiet = 1.0 / (2.0 * rate * T(b));
  if (iters_out) *iters_out = iters;
  const bool tight = bmem < e.bmax && b > 0.35 * bmax;
  // admission iterations: one per request (continuous), one per batch (static: drain, then admit)
  const double adm = e.stat ? n / std::max(1.0, b) : n;
  return 256.0 * iters + 22000.0 * adm + 13600.0 * n * (tight ? 1.0 : 0.0);
}

// The lean unified kernel runs one point per CTA with a helper warp (variant 0) when a run is
// latency-bound: at most kHelperPointsPerSm points per SM (a point's serial chain, not the SM's
// issue rate, then sets the kernel time: DESIGN.md §7).  TOKENSIM_HELPER=0/1 overrides (A/B).
constexpr u64 kHelperPointsPerSm = 4;
static bool helper_run(const tokensim_sweep *h, u64 n_run, int sm_count) {
  if (h->opt.topology == TOKENSIM_PD_PAIR) return false;
  if (!helper_fits(h->smem_per_warp(), h->nwords_max)) return false;
  if (const char *e = getenv("TOKENSIM_HELPER")) return atoi(e) != 0;
  // full kernel: at most 2 points per SM (c7, 256 points: 95 -> 79 ms; c8, 384: 17.1 -> 19.6)
  return n_run <= (h->full ? 2u : kHelperPointsPerSm) * (u64)sm_count;
}

// NVTX range for the enqueue of one run and of each launch (names appear in nsys / ncu --nvtx)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

static Layout make_layout(const tokensim_sweep *h, u64 n_run, int sm_count, int blocks_per_sm_limit) {
  Layout L{};
  const u64 n = h->n_slots();
  const u64 nconv = h->wl.num_requests;
  const bool mr = h->wl.multi_round != 0;
  const bool trace_mode = h->wl.len_dist == TOKENSIM_LEN_TRACE;
  const u64 groups = trace_mode ? 1 : (u64)h->rates.size() * h->seeds.size();
  L.n_run = n_run;
  const bool pd = h->opt.topology == TOKENSIM_PD_PAIR;
  const bool pair = pd && !h->pd_general;
  const size_t per_warp = h->smem_per_warp();
  u32 wpb = (u32)std::max<size_t>(1, std::min<size_t>(4, (227 * 1024) / per_warp));
  // fewer points than SMs x wpb: spread them one warp per SM first (each point is a serial
  // latency-bound chain; co-resident warps would only share the SM's LSU/MIO pipes)
  if (const char *e = getenv("TOKENSIM_WPB")) wpb = (u32)std::max(1, std::min(4, atoi(e)));
  else if ((u64)n_run <= (u64)sm_count || helper_run(h, n_run, sm_count)) wpb = 1;
  if (h->pd_general) wpb = 1;  // the node kernel: one point per CTA of pd_y warps
  // lean kernel without the helper, at most one wave of 8 warps per SM (4-8 points per SM): the
  // longest chains set the time, and 6 warps per SM (3 x 2 CTAs) run them faster than 8 (the
  // 2- and 4-GPU shards of C3 / C4: 222 -> 198 ms, 252 -> 237 ms)
  const bool six = !getenv("TOKENSIM_WPB") && !getenv("TOKENSIM_BPS") && !h->full && !pd &&
                   !helper_run(h, n_run, sm_count) && n_run > 4ull * (u64)sm_count && n_run <= 8ull * (u64)sm_count &&
                   wpb >= 3;
  if (six) wpb = 3;
  u32 bps = (u32)std::max<size_t>(1, (227 * 1024) / (per_warp * wpb));
  bps = std::min<u32>(bps, six ? 2u : 16u);
  if (blocks_per_sm_limit > 0) bps = std::min<u32>(bps, (u32)blocks_per_sm_limit);
  if (const char *e = getenv("TOKENSIM_BPS")) bps = std::min<u32>(bps, (u32)std::max(1, atoi(e)));  // A/B experiments
  const u64 need_warps = std::max<u64>(1, n_run);
  u64 blocks = std::min<u64>((u64)sm_count * bps, ceil_div(need_warps, wpb));
  L.wpb = wpb;
  L.blocks = (u32)std::max<u64>(1, blocks);
  L.warps_total = L.blocks * wpb;
  L.smem = per_warp * wpb;
  const u64 trace_cap = h->opt.trace_mode == TOKENSIM_TRACE_NONE ? 0 : h->opt.trace_cap_bytes / sizeof(tokensim_mem_sample);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align256(o + bytes);
    return at;
  };
  L.arrival = take(trace_mode ? 0 : groups * n * 8);
  L.prompt = take(trace_mode ? 0 : groups * n * 4);
  L.output = take(trace_mode ? 0 : groups * n * 4);
  L.rec = take(n_run * n * sizeof(tokensim_request_record));
  L.stats = take(n_run * sizeof(SimStats));
  L.trace = take(n_run * h->trace_nw() * trace_cap * sizeof(tokensim_mem_sample));
  L.itrec = take(n_run * (u64)h->opt.iteration_trace_cap * sizeof(tokensim_iter_record));
  L.summ = take(n_run * sizeof(tokensim_summary));
  L.bt = take((size_t)L.warps_total * h->bt_tables() * h->cap * h->bt_len * 4);
  L.order = take(n_run * 4 + 4);
  L.queue = take(256);
  L.sched = take((513 + 1024) * 4);
  L.scratch = take(n > kSummarySmemKeys ? n_run * n * 8 : 0);
  L.ring = take(pair ? (size_t)L.warps_total * h->max_total_blocks * 4 : 0);
  L.fifo = take(pair ? (size_t)L.warps_total * n * 32 : 0);
  L.pdn_per_warp = h->pd_general ? align256(pdn_global_per_warp(n, h->cap, h->bt_len, h->pd_x, h->pd_y)) : 0;
  L.pdn = take((size_t)L.warps_total * L.pdn_per_warp);
  L.mr_conv = take(mr ? groups * n * 4 : 0);
  L.mr_base = take(mr ? groups * nconv * 4 : 0);
  L.mr_nr = take(mr ? groups * nconv * 4 : 0);
  L.mr_ntot = take(mr ? groups * 4 : 0);
  L.mr_a0 = take(mr ? groups * nconv * 8 : 0);
  L.mr_p0 = take(mr ? groups * nconv * 4 : 0);
  L.mr_o0 = take(mr ? groups * nconv * 4 : 0);
  // per warp: arrival FIFO (rid u32 + time i64) x n, follow-up heap (time i64 + conv u32) x
  // nconv, next round / cached tokens / LRU prev / LRU next (u32) x nconv
  L.mr_per_warp = mr ? align256(n * 12 + nconv * 12 + nconv * 16 + 64) : 0;
  L.mr = take((size_t)L.warps_total * L.mr_per_warp);
  // the logs are per simulating warp: a node CTA has pd_y (+1 with the scheduler warp) of them
  const size_t log_warps = (size_t)L.warps_total * (h->pd_general ? h->pd_y + 1u : 1u);
  L.evlog = take(log_warps * 1024 * 16);
  L.itlog = take(log_warps * 256 * 64);
  // preload pipeline scratch of the helper-warp full kernel (layers + 1 doubles per warp)
  L.pipe_stride = h->opt.link_mode == TOKENSIM_LINK_PRELOAD ? ((size_t)h->model.num_layers + 1 + 31) & ~(size_t)31 : 0;
  L.pipe = take(log_warps * L.pipe_stride * 8);
  L.total = o;
  return L;
}

// SM count of `dev`; dev < 0: the largest over all visible devices (a workspace sized with it
// fits a run on any of them)
static int device_sms(int dev) {
  int sms = 148;
  int count = 0;
  if (cudaGetDeviceCount(&count) == cudaSuccess && count > 0) {
    if (dev >= 0) {
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
    } else {
      int best = 0;
      for (int d = 0; d < count; ++d) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) == cudaSuccess) best = std::max(best, v);
      }
      sms = best > 0 ? best : 148;
    }
  } else {
    cudaGetLastError();
  }
  return sms;
}

tokensim_status tokensim_sweep_workspace_size(const tokensim_sweep *h, uint64_t begin, uint64_t end,
                                              uint64_t stride, size_t *bytes) {
  if (!h || !bytes) return TOKENSIM_E_INVALID;
  if (!range_ok(h, begin, end, stride)) return TOKENSIM_E_RANGE;
  const Layout L = make_layout(h, count_run(begin, end, stride), device_sms(-1), 0);
  *bytes = L.total;
  return TOKENSIM_OK;
}

static tokensim_status upload_tables(tokensim_sweep *h, int dev) {
  if (h->d_tab && h->dev == dev) return TOKENSIM_OK;
  if (h->d_tab) {
    cudaSetDevice(h->dev);
    cudaFree(h->d_tab);
    h->d_tab = nullptr;
  }
  cudaSetDevice(dev);
  std::vector<char> blob;
  auto put = [&](const void *p, size_t bytes) {
    const size_t at = blob.size();
    blob.resize(align256(at + bytes));
    if (bytes) std::memcpy(blob.data() + at, p, bytes);
    return at;
  };
  h->off_hw = put(h->dhw.data(), h->dhw.size() * sizeof(DevHw));
  h->off_hp = put(h->dhp.data(), h->dhp.size() * sizeof(DevHP));
  h->off_pol = put(h->dpol.data(), h->dpol.size() * sizeof(DevPol));
  h->off_rates = put(h->rates.data(), h->rates.size() * sizeof(double));
  h->off_seeds = put(h->seeds.data(), h->seeds.size() * sizeof(uint64_t));
  h->off_pt = put(h->ptab.data(), h->ptab.size() * 4);
  h->off_ot = put(h->otab.data(), h->otab.size() * 4);
  h->off_tra = put(h->tr_a.data(), h->tr_a.size() * 8);
  h->off_trp = put(h->tr_p.data(), h->tr_p.size() * 4);
  h->off_tro = put(h->tr_o.data(), h->tr_o.size() * 4);
  cudaError_t e = cudaMalloc(&h->d_tab, blob.size());
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaMalloc(tables)");
  e = cudaMemcpy(h->d_tab, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaMemcpy(tables)");
  h->table_bytes_pending = blob.size();
  for (int i = 0; i < 4; ++i) {
    if (h->ev[i]) cudaEventDestroy(h->ev[i]);
    h->ev[i] = nullptr;
    e = cudaEventCreate(&h->ev[i]);
    if (e != cudaSuccess) return cuda_fail(h, e, "cudaEventCreate");
  }
  h->dev = dev;
  return TOKENSIM_OK;
}

tokensim_status tokensim_sweep_run(tokensim_sweep *h, int device, uint64_t begin, uint64_t end, uint64_t stride,
                                   void *d_workspace, size_t ws_bytes, void *cuda_stream) {
  if (!h) return TOKENSIM_E_INVALID;
  if (!range_ok(h, begin, end, stride)) return fail(h, TOKENSIM_E_RANGE, "run: bad point range");
  NvtxRange nv_run("tokensim_sweep_run");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(h, TOKENSIM_E_CUDA, "run: no CUDA device (there is no CPU fallback)");
  }
  if (device < 0 || device >= count) return fail(h, TOKENSIM_E_RANGE, "run: bad device index");
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaSetDevice");
  tokensim_status s = upload_tables(h, device);
  if (s != TOKENSIM_OK) return s;
  const u64 n_run = count_run(begin, end, stride);
  int sms = device_sms(device);
  const size_t per_warp = h->smem_per_warp();
  Layout L0 = make_layout(h, n_run, sms, 0);
  int occ = 0;
  const bool helper = L0.wpb == 1 && helper_run(h, n_run, sms);
  // extended stretches pay off while the chains have their SM nearly to themselves (<= 2 points
  // per SM: C4 at 8 GPUs 122 -> 115 ms) or have long quiet stretches; otherwise their hot code
  // costs more (C3 at 8 GPUs, ~4 per SM: 142 -> 162 ms).  TOKENSIM_XS=0/1 overrides (A/B).
  bool xs = n_run <= 4ull * (u64)sms;
  if (xs && helper && n_run > 0 && !h->wl.multi_round && h->wl.len_dist != TOKENSIM_LEN_TRACE) {
    // ... and only for chains with long quiet stretches: the median point's expected iterations
    // between events >= 6 (C1 27: 0.83 -> 0.78 ms with them; C2 1.9: 7.51 -> 7.80 ms without)
    std::vector<double> q(n_run);
    for (u64 j = 0; j < n_run; ++j) {
      const Coords c = decode_point(begin + j * stride, (u32)h->pol.size(), (u32)h->rates.size(),
                                    (u32)h->seeds.size());
      lpt_cost(h, (u32)((size_t)c.hw * h->pol.size() + c.pol), h->rates[c.rate], &q[j]);
    }
    std::nth_element(q.begin(), q.begin() + n_run / 2, q.end());
    // (2-4 points per SM: only for longer quiet stretches -- C4's 4-GPU shard, median 13.7:
    // 160 -> 143 ms with them; C3's 8-GPU shard, median 9.6: 151 -> 160 ms)
    xs = q[n_run / 2] >= (n_run <= 2ull * (u64)sms ? 6.0 : 12.0);
    if (getenv("TOKENSIM_DEBUG_XS")) fprintf(stderr, "tokensim: median quiet %.2f, %.2f points per SM\n", q[n_run / 2], (double)n_run / sms);
  }
  if (const char *ev = getenv("TOKENSIM_XS")) xs = atoi(ev) != 0;
  // (the node kernel's occupancy is asked for its CTA of pd_y warps)
  // node: the register-capped two-CTAs-per-SM build once there are more points than SMs
  bool node_two = h->pd_general && h->pd_y <= 6 && n_run > (u64)sms;
  if (const char *ev = getenv("TOKENSIM_NODE_TWO")) node_two = h->pd_general && h->pd_y <= 6 && atoi(ev) != 0;  // A/B
  // node, one wave: the scheduler on a warp of its own, alongside the decode phases
  bool node_sw = h->pd_general && !node_two && n_run <= (u64)sms;
  if (const char *ev = getenv("TOKENSIM_NODE_SW")) node_sw = h->pd_general && !node_two && atoi(ev) != 0;  // A/B
  e = sim_occupancy(sim_variant(h->full, h->opt.topology == TOKENSIM_PD_PAIR, h->pd_general, !helper, xs), (int)h->cap,
                    h->pd_general ? (int)h->pd_y + (node_sw ? 1 + 32 : 0) + (node_two ? 16 : 0) : (int)L0.wpb,
                    per_warp * L0.wpb, h->nwords_max,
                    &occ);
  if (e != cudaSuccess) return cuda_fail(h, e, "occupancy");
  if (occ < 1)
    return fail(h, TOKENSIM_E_NOMEM,
                "run: simulation kernel does not fit on an SM (" + std::to_string(per_warp) +
                    " B of shared memory per point" +
                    (h->pd_general ? std::string(", an xP:yD node keeps every decode worker's slots on chip: fewer decode "
                                                 "workers or max_num_seqs <= 256") : std::string()) + ")");
  const Layout L = make_layout(h, n_run, sms, occ);
  char *ws = static_cast<char *>(d_workspace);
  if (!ws) {
    if (h->owned_bytes < L.total) {
      if (h->owned_ws) cudaFree(h->owned_ws);
      h->owned_ws = nullptr;
      h->owned_bytes = 0;
      e = cudaMalloc(&h->owned_ws, L.total);
      if (e != cudaSuccess) return fail(h, TOKENSIM_E_NOMEM, std::string("cudaMalloc(workspace): ") + cudaGetErrorString(e));
      h->owned_bytes = L.total;
    }
    ws = h->owned_ws;
    ws_bytes = h->owned_bytes;
  }
  if (ws_bytes < L.total)
    return fail(h, TOKENSIM_E_NOMEM, "run: workspace too small: " + std::to_string(ws_bytes) + " < " + std::to_string(L.total));
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);

  SweepParams P{};
  P.M = h->M;
  {
    const DevModel &M = h->M;  // exact: every coefficient is an integer below 2^53 (validated at create)
    DevModelF &F = P.MF;
    F.h = (double)M.h;
    F.q2g = (double)M.q2g;
    F.hq2g = (double)M.hq2g;
    F.qh = (double)M.qh;
    F.q = (double)M.q;
    F.q4 = (double)(4 * M.q);
    F.hfu = (double)M.hfu;
    F.fu = (double)M.fu;
    F.fh = (double)M.fh;
    F.f = (double)M.f;
    F.Vh = (double)M.Vh;
    F.V = (double)M.V;
    F.s = (double)M.s;
    F.att_tok = (double)M.att_tok;
    F.g2 = (double)M.g2;
    F.L = (double)M.L;
    F.twoL = (double)(2 * M.L);
  }
  P.hw = reinterpret_cast<const DevHw *>(h->d_tab + h->off_hw);
  P.hp = reinterpret_cast<const DevHP *>(h->d_tab + h->off_hp);
  P.pol = reinterpret_cast<const DevPol *>(h->d_tab + h->off_pol);
  P.rates = reinterpret_cast<const double *>(h->d_tab + h->off_rates);
  P.seeds = reinterpret_cast<const u64 *>(h->d_tab + h->off_seeds);
  P.n_hw = h->n_hw_axis;
  P.n_pol = (u32)h->pol.size();
  P.n_rates = (u32)h->rates.size();
  P.n_seeds = (u32)h->seeds.size();
  P.topology = h->opt.topology;
  P.n_req = (u32)h->n_slots();
  const bool trace_mode = h->wl.len_dist == TOKENSIM_LEN_TRACE;
  P.len_dist = h->wl.len_dist == TOKENSIM_LEN_SHAREGPT_SYNTH_V1 ? (u32)TOKENSIM_LEN_TABLE : h->wl.len_dist;
  P.n_groups = trace_mode ? 0 : P.n_rates * P.n_seeds;
  P.prompt_a = h->wl.prompt_a;
  P.prompt_b = h->wl.prompt_b;
  P.output_a = h->wl.output_a;
  P.output_b = h->wl.output_b;
  P.pt = reinterpret_cast<const u32 *>(h->d_tab + h->off_pt);
  P.ot = reinterpret_cast<const u32 *>(h->d_tab + h->off_ot);
  if (trace_mode) {
    P.arrival = reinterpret_cast<i64 *>(h->d_tab + h->off_tra);
    P.prompt = reinterpret_cast<u32 *>(h->d_tab + h->off_trp);
    P.output = reinterpret_cast<u32 *>(h->d_tab + h->off_tro);
    P.group_of_point_mode = 1;
  } else {
    P.arrival = reinterpret_cast<i64 *>(ws + L.arrival);
    P.prompt = reinterpret_cast<u32 *>(ws + L.prompt);
    P.output = reinterpret_cast<u32 *>(ws + L.output);
    P.group_of_point_mode = 0;
  }
  P.begin = begin;
  P.stride = stride;
  P.n_run = n_run;
  P.order = reinterpret_cast<const u32 *>(ws + L.order);
  P.queue = reinterpret_cast<u32 *>(ws + L.queue);
  P.sched = reinterpret_cast<u32 *>(ws + L.sched);
  P.helper_mode = helper ? ((xs || h->full) ? 1u : 2u) : 0u;  // (the full helper kernel always has them)
  P.rec = reinterpret_cast<tokensim_request_record *>(ws + L.rec);
  P.stats = reinterpret_cast<SimStats *>(ws + L.stats);
  P.trace = reinterpret_cast<tokensim_mem_sample *>(ws + L.trace);
  P.trace_nw = h->trace_nw();
  P.bt_tables = h->bt_tables();
  P.trace_cap = h->opt.trace_mode == TOKENSIM_TRACE_NONE ? 0 : h->opt.trace_cap_bytes / sizeof(tokensim_mem_sample);
  P.itrec = reinterpret_cast<tokensim_iter_record *>(ws + L.itrec);
  P.it_cap = h->opt.iteration_trace_cap;
  P.summ = reinterpret_cast<tokensim_summary *>(ws + L.summ);
  P.bt = reinterpret_cast<u32 *>(ws + L.bt);
  P.bt_len = h->bt_len;
  P.cap_slots = h->cap;
  P.nwords_max = h->nwords_max;
  P.n_warps_total = L.warps_total;
  P.trace_mode = h->opt.trace_mode;
  P.bin_ns = h->opt.trace_bin_ns ? h->opt.trace_bin_ns : 1;
  P.horizon = h->opt.horizon_ns;
  P.slo_ttft_ns = (i64)std::floor(h->opt.slo_ttft_s * 1e9 + 0.5);
  P.slo_mtpot_ns = (i64)std::floor(h->opt.slo_mtpot_s * 1e9 + 0.5);
  P.pd_link_inv = h->opt.pd_link_bw > 0 ? 1.0 / h->opt.pd_link_bw : 0.0;
  P.scratch = reinterpret_cast<u64 *>(ws + L.scratch);
  P.ff_enable = (h->opt.flags & TOKENSIM_OPT_NO_FAST_FORWARD) ? 0u : 1u;
  P.pd_ring = reinterpret_cast<u32 *>(ws + L.ring);
  P.pd_ring_len = h->max_total_blocks ? h->max_total_blocks : 1;
  P.pd_fifo = reinterpret_cast<unsigned char *>(ws + L.fifo);
  P.pdn_scratch = reinterpret_cast<unsigned char *>(ws + L.pdn);
  P.pdn_bytes_per_warp = L.pdn_per_warp;
  P.pd_x = h->pd_x;
  P.pd_y = h->pd_y;
  P.node_two = node_two ? 1u : 0u;
  P.node_sw = node_sw ? 1u : 0u;
  P.dispatch = h->opt.dispatch;
  P.link_mode = h->opt.link_mode;
  P.preload_buf = h->opt.preload_buffer_bytes;
  P.multi_round = h->wl.multi_round ? 1u : 0u;
  P.memory_cache = h->opt.memory_cache ? 1u : 0u;
  P.n_conv = h->wl.num_requests;
  P.think_ns = h->wl.think_mean_s * 1e9;
  P.fetch_s = h->opt.cache_fetch_ns_per_block * 1e-9;
  P.cache_cap = h->opt.cache_capacity_blocks;
  P.mr_conv = reinterpret_cast<u32 *>(ws + L.mr_conv);
  P.mr_base = reinterpret_cast<u32 *>(ws + L.mr_base);
  P.mr_nr = reinterpret_cast<u32 *>(ws + L.mr_nr);
  P.mr_ntot = reinterpret_cast<u32 *>(ws + L.mr_ntot);
  P.mr_a0 = reinterpret_cast<i64 *>(ws + L.mr_a0);
  P.mr_p0 = reinterpret_cast<u32 *>(ws + L.mr_p0);
  P.mr_o0 = reinterpret_cast<u32 *>(ws + L.mr_o0);
  P.mr_scratch = reinterpret_cast<unsigned char *>(ws + L.mr);
  P.mr_bytes_per_warp = L.mr_per_warp;
  P.pd_general = h->pd_general ? 1u : 0u;
  P.full = h->full ? 1u : 0u;
  P.n_sms = (u32)sms;
  {
    bool p2 = true;  // the kernels specialise their block arithmetic to shifts and masks
    for (const auto &pl : h->pol) p2 = p2 && (pl.block_size & (pl.block_size - 1)) == 0;
    P.all_p2 = p2 ? 1u : 0u;
  }
  P.evlog = reinterpret_cast<uint4 *>(ws + L.evlog);
  P.itlog = reinterpret_cast<ulonglong2 *>(ws + L.itlog);
  P.pipe = reinterpret_cast<double *>(ws + L.pipe);
  P.pipe_stride = L.pipe_stride;

  // longest-estimated-first order (LPT): simulated span / per-iteration floor
  std::vector<u32> order(n_run + 1, 0);
  {
    std::vector<std::pair<double, u32>> est(n_run);
    for (u64 j = 0; j < n_run; ++j) {
      const Coords c = decode_point(begin + j * stride, P.n_pol, P.n_rates, P.n_seeds);
      const double span = (double)P.n_req / h->rates[c.rate];
      const u32 hwe = P.topology == TOKENSIM_PD_PAIR ? c.hw % P.n_hw : c.hw;  // decode worker dominates
      static const bool lpt_old = getenv("TOKENSIM_LPT_OLD") != nullptr;  // A/B: the round-1 estimate
      // the cost estimate orders throughput-bound runs (8 warps per SM); a latency-bound run (the
      // helper kernel) is set by its longest chains, which span / T(1) -- iterations -- ranks better
      // (C3 at 8 emulated GPUs: 142 ms by iterations, 163 ms by the cost estimate)
      const bool unified = !lpt_old && P.topology != TOKENSIM_PD_PAIR && !h->wl.multi_round && !trace_mode;
      static const int lpt_helper = getenv("TOKENSIM_LPT_HELPER") ? atoi(getenv("TOKENSIM_LPT_HELPER")) : 0;
      double est_j = span / h->est_T1[(size_t)hwe * P.n_pol + c.pol];
      if (unified && (!helper || lpt_helper)) {
        double it_j = 0;
        const double cst = lpt_cost(h, (u32)((size_t)hwe * P.n_pol + c.pol), h->rates[c.rate], nullptr, &it_j);
        est_j = !helper ? cst : lpt_helper == 1 ? it_j : cst;
      }
      est[j] = {est_j, (u32)j};
    }
    if (const char *df = getenv("TOKENSIM_LPT_DUMP")) {  // observability: the estimates, one double per run point
      if (FILE *f = fopen(df, "wb")) {
        for (u64 j = 0; j < n_run; ++j) fwrite(&est[j].first, 8, 1, f);
        fclose(f);
      }
    }
    if (const char *cf = getenv("TOKENSIM_LPT_COSTS")) {  // A/B experiments only: measured per-point costs
      if (FILE *f = fopen(cf, "rb")) {
        std::vector<double> c(h->n_points);
        if (fread(c.data(), 8, c.size(), f) == c.size())
          for (u64 j = 0; j < n_run; ++j) est[j].first = c[begin + j * stride];
        fclose(f);
      }
    }
    std::stable_sort(est.begin(), est.end(), [](const std::pair<double, u32> &a, const std::pair<double, u32> &b) {
      return a.first > b.first;
    });
    for (u64 j = 0; j < n_run; ++j) order[j] = est[j].second;
    // Heads (helper mode with more points than SMs): TOKENSIM_HEADS=K gives the K longest-
    // estimated points an SM each (the other CTAs on a head's SM leave).  Off by default: with
    // one CTA per point the leaving CTAs' share of the queue is serialised onto the others, and
    // C3 / C4 at 8 emulated GPUs measured slower for every K > 0.
    P.n_heads = 0;
    if (helper && n_run > (u64)sms)
      if (const char *ev = getenv("TOKENSIM_HEADS"))
        P.n_heads = (u32)std::min<long>(std::max(0, atoi(ev)), (long)std::min<u64>((u64)sms / 2, 1024));
  }
  e = cudaMemcpyAsync(ws + L.order, order.data(), (n_run + 1) * 4, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaMemcpyAsync(order)");
  e = cudaMemsetAsync(ws + L.queue, 0, 256, st);
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaMemsetAsync(queue)");
  e = cudaMemsetAsync(ws + L.sched, 0, (513 + 1024) * 4, st);
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaMemsetAsync(sched)");
  h->n_launches = 0;
  cudaEventRecord(h->ev[0], st);
  if (n_run > 0 && !trace_mode) {
    NvtxRange nv("tokensim.workload_kernel");
    e = launch_workload(P, st);
    if (e != cudaSuccess) return cuda_fail(h, e, "workload_kernel");
    ++h->n_launches;
  }
  cudaEventRecord(h->ev[1], st);
  if (n_run > 0) {
    NvtxRange nv("tokensim.sim_kernel");
    e = launch_sim(P, (int)h->cap, (int)L.wpb, (int)L.blocks, L.smem, st);
    if (e != cudaSuccess) return cuda_fail(h, e, "sim_kernel");
    ++h->n_launches;
  }
  cudaEventRecord(h->ev[2], st);
  if (n_run > 0) {
    NvtxRange nv("tokensim.summary_kernel");
    e = launch_summary(P, st);
    if (e != cudaSuccess) return cuda_fail(h, e, "summary_kernel");
    ++h->n_launches;
  }
  cudaEventRecord(h->ev[3], st);
  h->h2d_bytes = h->table_bytes_pending + (n_run + 1) * 4;
  h->table_bytes_pending = 0;
  // the host order buffer is pageable: the copy above is staged before return
  h->ran = true;
  h->begin = begin;
  h->end = end;
  h->stride = stride;
  h->n_run = n_run;
  h->ws = ws;
  h->ws_bytes = ws_bytes;
  h->stream = st;
  h->P = P;
  h->lay = L;
  return TOKENSIM_OK;
}

static tokensim_status local_index(const tokensim_sweep *h, u64 point, u64 *j) {
  if (point >= h->n_points) return TOKENSIM_E_RANGE;
  if (!h->ran || point < h->begin || point >= h->end || (point - h->begin) % h->stride) return TOKENSIM_E_STATE;
  *j = (point - h->begin) / h->stride;
  return TOKENSIM_OK;
}

static tokensim_status sync_run(tokensim_sweep *h) {
  cudaSetDevice(h->dev);
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "stream");
  return TOKENSIM_OK;
}

static tokensim_status copy_d2h(tokensim_sweep *h, void *dst, const void *src, size_t bytes) {
  if (!bytes) return TOKENSIM_OK;
  cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaMemcpy D2H");
  return TOKENSIM_OK;
}

tokensim_status tokensim_get_summary(const tokensim_sweep *hc, uint64_t point, tokensim_summary *out) {
  tokensim_sweep *h = const_cast<tokensim_sweep *>(hc);
  if (!h || !out) return TOKENSIM_E_INVALID;
  u64 j;
  tokensim_status s = local_index(h, point, &j);
  if (s == TOKENSIM_E_STATE && point < h->imported.size() && h->imported[point].version) {
    *out = h->imported[point];
    return TOKENSIM_OK;
  }
  if (s != TOKENSIM_OK) return fail(h, s, "get_summary: point not run by this handle");
  if ((s = sync_run(h)) != TOKENSIM_OK) return s;
  return copy_d2h(h, out, h->P.summ + j, sizeof(tokensim_summary));
}

tokensim_status tokensim_get_summaries(const tokensim_sweep *hc, tokensim_summary *out, uint64_t capacity,
                                       uint64_t *n_out) {
  tokensim_sweep *h = const_cast<tokensim_sweep *>(hc);
  if (!h || !n_out) return TOKENSIM_E_INVALID;
  if (!h->ran) return fail(h, TOKENSIM_E_STATE, "get_summaries: no run");
  *n_out = h->n_run;
  if (!out || capacity == 0) return TOKENSIM_OK;
  if (capacity < h->n_run) return TOKENSIM_E_TRUNCATED;
  tokensim_status s = sync_run(h);
  if (s != TOKENSIM_OK) return s;
  return copy_d2h(h, out, h->P.summ, h->n_run * sizeof(tokensim_summary));
}

tokensim_status tokensim_get_summaries_device(const tokensim_sweep *h, const void **d_ptr, size_t *bytes) {
  if (!h || !d_ptr || !bytes) return TOKENSIM_E_INVALID;
  if (!h->ran) return TOKENSIM_E_STATE;
  *d_ptr = h->P.summ;
  *bytes = h->n_run * sizeof(tokensim_summary);
  return TOKENSIM_OK;
}

tokensim_status tokensim_import_summaries(tokensim_sweep *h, const void *host_ptr, size_t bytes) {
  if (!h || (!host_ptr && bytes)) return TOKENSIM_E_INVALID;
  if (bytes % sizeof(tokensim_summary)) return fail(h, TOKENSIM_E_INVALID, "import_summaries: bytes % 384 != 0");
  const tokensim_summary *s = static_cast<const tokensim_summary *>(host_ptr);
  if (h->imported.size() < h->n_points) h->imported.resize(h->n_points);
  for (size_t i = 0; i < bytes / sizeof(tokensim_summary); ++i) {
    if (!s[i].version) continue;
    if (s[i].point >= h->n_points) return fail(h, TOKENSIM_E_RANGE, "import_summaries: point out of range");
    h->imported[s[i].point] = s[i];
  }
  return TOKENSIM_OK;
}

tokensim_status tokensim_get_request_records(const tokensim_sweep *hc, uint64_t point, tokensim_request_record *out,
                                             uint64_t capacity, uint64_t *n_out) {
  tokensim_sweep *h = const_cast<tokensim_sweep *>(hc);
  if (!h || !n_out) return TOKENSIM_E_INVALID;
  u64 j;
  tokensim_status s = local_index(h, point, &j);
  if (s != TOKENSIM_OK) return fail(h, s, "get_request_records: point not run by this handle");
  const u64 stride = h->n_slots();
  u64 n = stride;
  if (h->wl.multi_round) {  // this point's requests (rounds of its conversations)
    if ((s = sync_run(h)) != TOKENSIM_OK) return s;
    SimStats st;
    if ((s = copy_d2h(h, &st, h->P.stats + j, sizeof st)) != TOKENSIM_OK) return s;
    n = st.n_req;
  }
  *n_out = n;
  if (!out || capacity == 0) return TOKENSIM_OK;
  if (capacity < n) return TOKENSIM_E_TRUNCATED;
  if ((s = sync_run(h)) != TOKENSIM_OK) return s;
  return copy_d2h(h, out, h->P.rec + j * stride, n * sizeof(tokensim_request_record));
}

tokensim_status tokensim_get_iteration_trace(const tokensim_sweep *hc, uint64_t point, tokensim_iter_record *out,
                                             uint64_t capacity, uint64_t *n_out) {
  tokensim_sweep *h = const_cast<tokensim_sweep *>(hc);
  if (!h || !n_out) return TOKENSIM_E_INVALID;
  u64 j;
  tokensim_status s = local_index(h, point, &j);
  if (s != TOKENSIM_OK) return fail(h, s, "get_iteration_trace: point not run by this handle");
  if (h->opt.iteration_trace_cap == 0) return fail(h, TOKENSIM_E_STATE, "iteration trace disabled (iteration_trace_cap = 0)");
  if ((s = sync_run(h)) != TOKENSIM_OK) return s;
  SimStats st;
  if ((s = copy_d2h(h, &st, h->P.stats + j, sizeof st)) != TOKENSIM_OK) return s;
  *n_out = st.iter_n;
  if (!out || capacity == 0) return TOKENSIM_OK;
  if (capacity < st.iter_n) return TOKENSIM_E_TRUNCATED;
  return copy_d2h(h, out, h->P.itrec + j * h->P.it_cap, st.iter_n * sizeof(tokensim_iter_record));
}

// Decoder of the compressed FULL memory trace (trace_codec.cuh; format in include/tokensim.h):
// three LEB128 varints per iteration -- idle gap, zigzag dT, zigzag dblocks.  Rebuilds the
// documented FULL samples (t_start, T, blocks * T, blocks, 1).  false: the stream is malformed.
static bool read_varint(const unsigned char *&p, const unsigned char *end, u64 &x) {
  x = 0;
  for (u32 sh = 0; sh < 64; sh += 7) {
    if (p == end) return false;
    const unsigned char b = *p++;
    x |= (u64)(b & 0x7fu) << sh;
    if (!(b & 0x80u)) return true;
  }
  return false;
}
static i64 unzigzag(u64 z) { return (i64)(z >> 1) ^ -(i64)(z & 1u); }
static bool decode_full_trace(const unsigned char *buf, size_t bytes, u64 n, tokensim_mem_sample *out) {
  const unsigned char *p = buf, *end = buf + bytes;
  i64 te = 0, T = 0, blk = 0;
  for (u64 k = 0; k < n; ++k) {
    u64 gap, dT, dB;
    if (!read_varint(p, end, gap) || !read_varint(p, end, dT) || !read_varint(p, end, dB)) return false;
    const i64 ts = te + (i64)gap;
    T += unzigzag(dT);
    blk += unzigzag(dB);
    if (T < 0 || blk < 0 || blk > 0xffffffffll) return false;
    te = ts + T;
    tokensim_mem_sample &sm = out[k];
    sm.t_ns = ts;
    sm.dur_ns = T;
    sm.block_ns = (u64)blk * (u64)T;
    sm.blocks_max = (u32)blk;
    sm.n_iter = 1;
  }
  return p == end;
}

tokensim_status tokensim_get_mem_trace(const tokensim_sweep *hc, uint64_t point, uint32_t worker,
                                       tokensim_mem_sample *out, uint64_t capacity, uint64_t *n_out) {
  tokensim_sweep *h = const_cast<tokensim_sweep *>(hc);
  if (!h || !n_out) return TOKENSIM_E_INVALID;
  const u32 n_workers = h->opt.topology == TOKENSIM_PD_PAIR ? h->pd_x + h->pd_y : 1u;
  if (worker >= n_workers) return TOKENSIM_E_RANGE;
  u64 j;
  tokensim_status s = local_index(h, point, &j);
  if (s != TOKENSIM_OK) return fail(h, s, "get_mem_trace: point not run by this handle");
  if (h->opt.trace_mode == TOKENSIM_TRACE_NONE) return fail(h, TOKENSIM_E_STATE, "memory trace disabled");
  if ((s = sync_run(h)) != TOKENSIM_OK) return s;
  SimStats st;
  if ((s = copy_d2h(h, &st, h->P.stats + j, sizeof st)) != TOKENSIM_OK) return s;
  const u64 cnt = st.trace_n[worker];
  *n_out = cnt;
  if (!out || capacity == 0) return TOKENSIM_OK;
  if (capacity < cnt) return TOKENSIM_E_TRUNCATED;
  const tokensim_mem_sample *src = h->P.trace + (j * h->P.trace_nw + worker) * h->P.trace_cap;
  if (h->opt.trace_mode == TOKENSIM_TRACE_FULL) {
    // the compressed stream (trace_codec.cuh): decode it here into one sample per iteration
    std::vector<unsigned char> buf(st.trace_b[worker]);
    if (!buf.empty() && (s = copy_d2h(h, buf.data(), src, buf.size())) != TOKENSIM_OK) return s;
    if (!decode_full_trace(buf.data(), buf.size(), cnt, out))
      return fail(h, TOKENSIM_E_STATE, "get_mem_trace: corrupt FULL trace stream");
  } else {
    s = copy_d2h(h, out, src, cnt * sizeof(tokensim_mem_sample));
    if (s != TOKENSIM_OK) return s;
  }
  return (st.flags & TOKENSIM_PT_TRACE_OVERFLOW) ? TOKENSIM_E_OVERFLOW : TOKENSIM_OK;
}

tokensim_status tokensim_get_mem_trace_encoded(const tokensim_sweep *hc, uint64_t point, uint32_t worker,
                                               uint8_t *out, uint64_t capacity, uint64_t *n_bytes,
                                               uint64_t *n_samples) {
  tokensim_sweep *h = const_cast<tokensim_sweep *>(hc);
  if (!h || !n_bytes) return TOKENSIM_E_INVALID;
  const u32 n_workers = h->opt.topology == TOKENSIM_PD_PAIR ? h->pd_x + h->pd_y : 1u;
  if (worker >= n_workers) return TOKENSIM_E_RANGE;
  u64 j;
  tokensim_status s = local_index(h, point, &j);
  if (s != TOKENSIM_OK) return fail(h, s, "get_mem_trace_encoded: point not run by this handle");
  if (h->opt.trace_mode != TOKENSIM_TRACE_FULL) return fail(h, TOKENSIM_E_STATE, "get_mem_trace_encoded: FULL trace mode only");
  if ((s = sync_run(h)) != TOKENSIM_OK) return s;
  SimStats st;
  if ((s = copy_d2h(h, &st, h->P.stats + j, sizeof st)) != TOKENSIM_OK) return s;
  *n_bytes = st.trace_b[worker];
  if (n_samples) *n_samples = st.trace_n[worker];
  if (!out || capacity == 0) return TOKENSIM_OK;
  if (capacity < st.trace_b[worker]) return TOKENSIM_E_TRUNCATED;
  if (st.trace_b[worker] &&
      (s = copy_d2h(h, out, h->P.trace + (j * h->P.trace_nw + worker) * h->P.trace_cap, st.trace_b[worker])) != TOKENSIM_OK)
    return s;
  return (st.flags & TOKENSIM_PT_TRACE_OVERFLOW) ? TOKENSIM_E_OVERFLOW : TOKENSIM_OK;
}

tokensim_status tokensim_get_latency_quantiles(const tokensim_sweep *hc, uint64_t point, uint32_t metric,
                                               const uint32_t *q_bp, uint32_t n_q, double *out_seconds) {
  tokensim_sweep *h = const_cast<tokensim_sweep *>(hc);
  if (!h || (!q_bp && n_q) || (!out_seconds && n_q)) return TOKENSIM_E_INVALID;
  if (metric > TOKENSIM_MTPOT) return fail(h, TOKENSIM_E_RANGE, "get_latency_quantiles: metric out of range");
  for (u32 i = 0; i < n_q; ++i)
    if (q_bp[i] > 10000) return fail(h, TOKENSIM_E_RANGE, "get_latency_quantiles: q_bp must be in [0, 10000]");
  if (n_q == 0) return TOKENSIM_OK;
  u64 j;
  tokensim_status s = local_index(h, point, &j);
  if (s == TOKENSIM_E_STATE && point < h->imported.size() && h->imported[point].version) {
    for (u32 i = 0; i < n_q; ++i) {
      const int col = q_bp[i] == 5000 ? 0 : q_bp[i] == 9000 ? 1 : q_bp[i] == 9900 ? 2 : q_bp[i] == 10000 ? 3 : -1;
      if (col < 0) return fail(h, TOKENSIM_E_STATE, "get_latency_quantiles: only P50/P90/P99/max are available for points run elsewhere");
      out_seconds[i] = h->imported[point].stat[metric][col];
    }
    return TOKENSIM_OK;
  }
  if (s != TOKENSIM_OK) return fail(h, s, "get_latency_quantiles: point not run by this handle");
  if ((s = sync_run(h)) != TOKENSIM_OK) return s;
  const u64 n = h->n_slots();
  char *buf = nullptr;
  const size_t bytes = align256(n_q * 4) + align256(n_q * 8) + n * 8;
  cudaError_t e = cudaMalloc(&buf, bytes);
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaMalloc(quantiles)");
  u32 *d_q = reinterpret_cast<u32 *>(buf);
  double *d_out = reinterpret_cast<double *>(buf + align256(n_q * 4));
  u64 *d_keys = reinterpret_cast<u64 *>(buf + align256(n_q * 4) + align256(n_q * 8));
  e = cudaMemcpy(d_q, q_bp, n_q * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_quantiles(h->P, j, metric, d_q, n_q, d_out, d_keys, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e == cudaSuccess) e = cudaMemcpy(out_seconds, d_out, n_q * 8, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (e != cudaSuccess) return cuda_fail(h, e, "quantile_kernel");
  return TOKENSIM_OK;
}

tokensim_status tokensim_get_workload(const tokensim_sweep *hc, uint64_t point, int64_t *arrival_ns,
                                      uint32_t *prompt, uint32_t *output, uint64_t capacity) {
  tokensim_sweep *h = const_cast<tokensim_sweep *>(hc);
  if (!h) return TOKENSIM_E_INVALID;
  u64 j;
  tokensim_status s = local_index(h, point, &j);
  if (s != TOKENSIM_OK) return fail(h, s, "get_workload: point not run by this handle");
  const u64 n = h->n_slots();  // multi-round: per request, arrival = round 0 time or think gap
  if (capacity < n) return TOKENSIM_E_TRUNCATED;
  if ((s = sync_run(h)) != TOKENSIM_OK) return s;
  const Coords c = decode_point(point, h->P.n_pol, h->P.n_rates, h->P.n_seeds);
  const u64 g = h->P.group_of_point_mode ? 0 : (u64)c.rate * h->P.n_seeds + c.seed;
  if (arrival_ns && (s = copy_d2h(h, arrival_ns, h->P.arrival + g * n, n * 8)) != TOKENSIM_OK) return s;
  if (prompt && (s = copy_d2h(h, prompt, h->P.prompt + g * n, n * 4)) != TOKENSIM_OK) return s;
  if (output && (s = copy_d2h(h, output, h->P.output + g * n, n * 4)) != TOKENSIM_OK) return s;
  return TOKENSIM_OK;
}

tokensim_status tokensim_get_point_profile(const tokensim_sweep *hc, uint64_t point, tokensim_point_profile *out) {
  tokensim_sweep *h = const_cast<tokensim_sweep *>(hc);
  if (!h || !out) return TOKENSIM_E_INVALID;
  u64 j;
  tokensim_status s = local_index(h, point, &j);
  if (s != TOKENSIM_OK) return fail(h, s, "get_point_profile: point not run by this handle");
  if ((s = sync_run(h)) != TOKENSIM_OK) return s;
  SimStats st;
  if ((s = copy_d2h(h, &st, h->P.stats + j, sizeof st)) != TOKENSIM_OK) return s;
  out->n_iterations = st.n_iterations;
  out->ff_iterations = st.ff_iters;
  out->ff_stretches = st.ff_runs;
  out->sm_cycles = st.cycles;
  out->cycles_ff = st.cyc_ff;
  out->cycles_ff_failed = st.cyc_ff_fail;
  out->cycles_normal = st.cyc_normal;
  out->n_transfers = st.n_transfers;
  out->transfer_bytes = st.transfer_bytes;
  for (int q = 0; q < 8; ++q) out->normal_phase_cycles[q] = st.nphase[q];
  for (int q = 0; q < 8; ++q) out->stretch_phase_cycles[q] = st.phase[q];
  for (int q = 0; q < 5; ++q) out->ff_failed[q] = st.ff_fail[q];
  for (int q = 0; q < 5; ++q) out->ff_cut[q] = st.ff_cut[q];
  return TOKENSIM_OK;
}

tokensim_status tokensim_get_run_info(const tokensim_sweep *hc, tokensim_run_info *out) {
  tokensim_sweep *h = const_cast<tokensim_sweep *>(hc);
  if (!h || !out) return TOKENSIM_E_INVALID;
  if (!h->ran) return fail(h, TOKENSIM_E_STATE, "get_run_info: no run");
  tokensim_status s = sync_run(h);
  if (s != TOKENSIM_OK) return s;
  float ms[3] = {0, 0, 0};
  for (int i = 0; i < 3; ++i) {
    cudaError_t e = cudaEventElapsedTime(&ms[i], h->ev[i], h->ev[i + 1]);
    if (e != cudaSuccess) return cuda_fail(h, e, "cudaEventElapsedTime");
  }
  out->ms_workload = ms[0];
  out->ms_sim = ms[1];
  out->ms_summary = ms[2];
  out->n_launches = h->n_launches;
  out->sim_blocks = h->lay.blocks;
  out->sim_warps_per_block = h->lay.wpb;
  out->smem_per_warp = (u32)h->smem_per_warp();
  out->n_run = h->n_run;
  out->h2d_bytes = h->h2d_bytes;
  out->workspace_bytes = h->lay.total;
  out->helper_mode = h->P.helper_mode;
  out->n_heads = h->P.n_heads;
  return TOKENSIM_OK;
}

void tokensim_sweep_destroy(tokensim_sweep *h) {
  if (!h) return;
  if (h->dev >= 0) cudaSetDevice(h->dev);
  for (int i = 0; i < 4; ++i)
    if (h->ev[i]) cudaEventDestroy(h->ev[i]);
  if (h->d_tab) cudaFree(h->d_tab);
  if (h->owned_ws) cudaFree(h->owned_ws);
  delete h;
}

}  // extern "C"
