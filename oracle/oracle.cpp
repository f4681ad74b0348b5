// oracle.cpp -- the CPU ORACLE for TokenSim's batched design-space sweep.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no code,
// header, table or constant generator with the CUDA path (paper_2503_08415_b200/),
// and it imports nothing from it.
//
// What it is: a plain, slow, single-threaded simulation of ONE sweep point,
// written as the algorithm of SURVEY.md §8(c) step by step (c.1 derived
// constants, c.2 workload, c.4 iteration loop, c.5 cost table, c.6 metrics and
// digests), using std::set / std::vector and explicit per-request block lists.
// No blocking, fusion, incremental aggregates or reordering: every quantity is
// recomputed from its definition when it is needed.
//
// Paper anchors (PAPER.md line numbers): iteration-level scheduling with the
// default end-of-iteration breakpoint P:243; continuous vs static batching
// P:166-169; PagedAttention blocks P:172-173; preemption by moving
// KV to host P:456-457; max-memory-ratio admission P:460; compute
// simulator returning iteration time P:216 with prefill compute-bound / decode
// memory-bound P:160-161; latency percentiles P:321; TTFT and mTPOT SLOs
// P:458-465; memory footprint over time P:552-565.  Every reading of an
// ambiguous passage is listed in DESIGN.md ("Readings").
//
// Build: g++ -std=c++17 -O2 -ffp-contract=off -fPIC -shared (no -ffast-math).
// Every fp64 expression is evaluated in the order written in SURVEY §8(c).

#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <list>
#include <map>
#include <set>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;

bool fail(const std::string &m) {
  g_err = m;
  return false;
}

// ----------------------------------------------------------------- c.2 Philox4x32-10
// Random123 / cuRAND definition: 10 rounds, multipliers 0xD2511F53, 0xCD9E8D57,
// Weyl key increments 0x9E3779B9, 0xBB67AE85; round output
// {hi1^c1^k0, lo1, hi0^c3^k1, lo0}.
void philox(const u32 ctr_in[4], const u32 key_in[2], u32 out[4]) {
  u32 c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  u32 k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    u64 p0 = (u64)0xD2511F53u * (u64)c[0];
    u64 p1 = (u64)0xCD9E8D57u * (u64)c[2];
    u32 hi0 = (u32)(p0 >> 32), lo0 = (u32)p0;
    u32 hi1 = (u32)(p1 >> 32), lo1 = (u32)p1;
    u32 n[4] = {hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0};
    c[0] = n[0]; c[1] = n[1]; c[2] = n[2]; c[3] = n[3];
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

// ----------------------------------------------------------------- c.2 det_log
// ln(u) = e*ln2 + ln(m), ln(m) = 2*atanh(s), s = (m-1)/(m+1), atanh by its
// series in z = s^2 (13 terms, c_k = 1/(2k+1)) -- only + - * / and frexp.
double det_log(double u) {
  int e = 0;
  double m = std::frexp(u, &e);
  if (m < 0x1.6a09e667f3bcdp-1) {
    m = m * 2.0;
    e = e - 1;
  }
  double s = (m - 1.0) / (m + 1.0);
  double z = s * s;
  double p = 1.0 / 25.0;  // c_12
  for (int k = 11; k >= 0; --k) {
    double pz = p * z;
    p = pz + 1.0 / (double)(2 * k + 1);
  }
  const double LN2 = 0x1.62e42fefa39efp-1;
  double a = (double)e * LN2;
  double b = (2.0 * s) * p;
  return a + b;
}

// ----------------------------------------------------------------- c.6 digests
u64 mix(u64 x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
u64 fold(std::initializer_list<u64> f) {
  u64 h = 0x9E3779B97F4A7C15ull;
  for (u64 v : f) h = mix(h ^ v);
  return h;
}

u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }

// c.6 digests (our own verification device, not a paper quantity): a block event folds
// (k | kind << 48, id | block << 32); an iteration folds (k | worker << 40, t, T, N_p, C_d, blocks,
// S_p | D << 16 | m << 32 | n_res << 48, n_adm | n_fin << 16 | n_rej << 32).
u64 fold_block(u64 k, u64 kind, u64 id, u64 b) { return fold({k | (kind << 48), id | (b << 32)}); }
u64 fold_sched(u64 kw, u64 t, u64 T, u64 Sp, u64 D, u64 Np, u64 Cd, u64 m, u64 nres, u64 nadm, u64 nrej, u64 nfin,
               u64 blocks) {
  return fold({kw, t, T, Np, Cd, blocks, Sp | (D << 16) | (m << 32) | (nres << 48), nadm | (nfin << 16) | (nrej << 32)});
}

// ----------------------------------------------------------------- per-worker profile
struct Profile {
  double peak_flops, mem_bw, eff_flops, eff_bw;
  u64 mem_capacity;
  double reserve_frac, iter_overhead_s, host_link_bw;
  u32 tp_degree;
  double tp_link_bw;
  u64 kv_blocks_override;
};

Profile profile_of(const oracle_cfg &c, int decode_worker) {
  Profile p;
  if (!decode_worker) {
    p = {c.peak_flops, c.mem_bw, c.eff_flops, c.eff_bw, c.mem_capacity, c.reserve_frac,
         c.iter_overhead_s, c.host_link_bw, c.tp_degree, c.tp_link_bw, c.kv_blocks_override};
  } else {
    p = {c.d_peak_flops, c.d_mem_bw, c.d_eff_flops, c.d_eff_bw, c.d_mem_capacity,
         c.d_reserve_frac, c.d_iter_overhead_s, c.d_host_link_bw, c.d_tp_degree,
         c.d_tp_link_bw, c.d_kv_blocks_override};
  }
  return p;
}

// ----------------------------------------------------------------- c.1 derived constants
bool derive(const oracle_cfg &c, int decode_worker, oracle_derived &d) {
  const Profile pr = profile_of(c, decode_worker);
  const u64 s = c.dtype_bytes, L = c.L, h = c.h, V = c.vocab, f = c.ffn;
  const u64 q = (u64)c.n_heads * c.head_dim;
  const u64 g = (u64)c.n_kv * c.head_dim;
  // W = s*[ L*(h*(q+2g) + q*h + (gated?3:2)*h*f) + (tied?1:2)*V*h + (2L+1)*h ]
  const u64 per_layer = h * (q + 2 * g) + q * h + (c.gated ? 3 : 2) * h * f;
  d.W = s * (L * per_layer + (c.tied ? 1 : 2) * V * h + (2 * L + 1) * h);
  d.kvb = 2 * L * g * s;
  d.block_bytes = (u64)c.block_size * d.kvb;
  d.reserve = (u64)std::floor((double)pr.mem_capacity * pr.reserve_frac);
  if (pr.kv_blocks_override) {
    d.total_blocks = pr.kv_blocks_override;
  } else {
    if (pr.mem_capacity < d.W + d.reserve)
      return fail("mem_capacity " + std::to_string(pr.mem_capacity) + " < weights " +
                  std::to_string(d.W) + " + reserve " + std::to_string(d.reserve));
    d.total_blocks = (pr.mem_capacity - d.W - d.reserve) / d.block_bytes;
  }
  d.ratio_limit = (u64)std::floor(c.max_mem_ratio * (double)d.total_blocks);
  d.invF = 1.0 / (pr.peak_flops * pr.eff_flops);
  d.invB = 1.0 / (pr.mem_bw * pr.eff_bw);
  d.invH = 1.0 / pr.host_link_bw;
  d.invT = 1.0 / ((double)pr.tp_degree * pr.tp_link_bw);
  d.scale_ns = 1e9 / c.rate;
  d.slo_ttft_ns = (i64)std::floor(c.slo_ttft_s * 1e9 + 0.5);
  d.slo_mtpot_ns = (i64)std::floor(c.slo_mtpot_s * 1e9 + 0.5);
  return true;
}

// ----------------------------------------------------------------- c.2 workload
u32 table_draw(u32 n, const u32 *lo, const u32 *hi, const u32 *thr, u32 x, u32 y) {
  u32 b = n - 1;  // last bucket takes the rest
  for (u32 i = 0; i + 1 < n; ++i) {
    if (x < thr[i]) {
      b = i;
      break;
    }
  }
  return lo[b] + (u32)(((u64)y * (u64)(hi[b] - lo[b])) >> 32);
}

bool workload(const oracle_cfg &c, std::vector<i64> &a, std::vector<u32> &p, std::vector<u32> &o) {
  const u32 n = c.num_requests;
  a.assign(n, 0);
  p.assign(n, 0);
  o.assign(n, 0);
  if (c.len_dist == OR_LEN_TRACE) {
    for (u32 i = 0; i < n; ++i) {
      a[i] = c.trace_arrival_ns[i];
      p[i] = c.trace_prompt[i];
      o[i] = c.trace_output[i];
    }
    return true;
  }
  const u32 key[2] = {(u32)(c.seed & 0xffffffffu), (u32)(c.seed >> 32)};
  const double scale_ns = 1e9 / c.rate;
  i64 acc = 0;
  for (u32 i = 0; i < n; ++i) {
    const u32 cx[4] = {i, 0, 0, 0}, cy[4] = {i, 1, 0, 0};
    u32 X[4], Y[4];
    philox(cx, key, X);
    philox(cy, key, Y);
    const u64 v = ((u64)X[0] << 21) | (u64)(X[1] >> 11);
    const double u = (double)(v + 1) * 0x1p-53;
    const double E = -det_log(u);
    const double es = E * scale_ns;
    const i64 gap = (i64)std::floor(es + 0.5);
    acc += gap;
    a[i] = acc;
    u32 pl = 0, ol = 0;
    if (c.len_dist == OR_LEN_FIXED) {
      pl = c.prompt_a;
      ol = c.output_a;
    } else if (c.len_dist == OR_LEN_UNIFORM) {
      pl = c.prompt_a + (u32)(((u64)X[2] * (u64)(c.prompt_b - c.prompt_a + 1)) >> 32);
      ol = c.output_a + (u32)(((u64)Y[0] * (u64)(c.output_b - c.output_a + 1)) >> 32);
    } else if (c.len_dist == OR_LEN_TABLE) {
      pl = table_draw(c.pt_n, c.pt_lo, c.pt_hi, c.pt_thr, X[2], X[3]);
      ol = table_draw(c.ot_n, c.ot_lo, c.ot_hi, c.ot_thr, Y[0], Y[1]);
    } else {
      return fail("unknown len_dist");
    }
    if (ol > c.max_model_len - pl) ol = c.max_model_len - pl;  // o = min(o, mml - p)
    p[i] = pl;
    o[i] = ol;
  }
  return true;
}

// ----------------------------------------------------------------- c.5 cost model
struct Prefill {
  u64 P, c0;          // P new tokens after c0 already-computed ones (c0 > 0: a later chunk)
  bool emits = true;  // the entry samples a token (false for a non-final chunk, reading R-N3b)
};

struct CostCtx {
  u64 L, h, q, g, f, fu, V, s;
  double invF, invB, invH, invT, overhead;
  u32 tp;
  u32 link_mode;    // OR_LINK_SEQUENTIAL (A10) | OR_LINK_PRELOAD (NEXT-4)
  u64 preload_buf;  // PRELOAD buffer bytes
};

// NEXT-4 preload-buffer pipeline (reading R-N4): n chunks; the producer
// (the link) loads chunk i in `a` seconds once it has loaded chunk i-1 and a buffer slot is free
// (the consumer has taken chunk i-K); the consumer takes chunk i at S_i = max(C_{i-1}, P_i) and
// finishes it `b` later.  Returns C_n, the time the consumer finishes the last chunk.
double pipeline(u64 n, double a, double b, u64 K) {
  std::vector<double> P(n + 1, 0.0), S(n + 1, 0.0), C(n + 1, 0.0);
  for (u64 i = 1; i <= n; ++i) {
    double ready = P[i - 1];
    if (i > K) ready = std::fmax(ready, S[i - K]);
    P[i] = ready + a;
    S[i] = std::fmax(C[i - 1], P[i]);
    C[i] = S[i] + b;
  }
  return C[n];
}

CostCtx cost_ctx(const oracle_cfg &c, const oracle_derived &d, int decode_worker) {
  const Profile pr = profile_of(c, decode_worker);
  CostCtx k;
  k.L = c.L;
  k.h = c.h;
  k.q = (u64)c.n_heads * c.head_dim;
  k.g = (u64)c.n_kv * c.head_dim;
  k.f = c.ffn;
  k.fu = c.gated ? 2 * (u64)c.ffn : (u64)c.ffn;
  k.V = c.vocab;
  k.s = c.dtype_bytes;
  k.invF = d.invF;
  k.invB = d.invB;
  k.invH = d.invH;
  k.invT = d.invT;
  k.overhead = pr.iter_overhead_s;
  k.tp = pr.tp_degree;
  k.link_mode = c.link_mode;
  k.preload_buf = c.preload_buffer_bytes;
  return k;
}

i64 iter_time(const CostCtx &K, const std::vector<Prefill> &pf, const std::vector<u64> &dec,
              u64 swap_out, u64 swap_in = 0, u64 fetch_blocks = 0, double fetch_s = 0.0) {
  u64 Np = 0, Ap = 0, Kp = 0, Cd = 0, Sp = 0;
  const u64 D = dec.size();
  for (const Prefill &e : pf) {
    Np += e.P;
    Ap += e.P * e.c0 + e.P * (e.P + 1) / 2;
    Kp += e.c0 + e.P;
    Sp += e.emits ? 1 : 0;  // LM head rows: entries that sample a token
  }
  for (u64 c : dec) Cd += c;
  const u64 N = Np + D, S = Sp + D;
  const u64 h = K.h, q = K.q, g = K.g, f = K.f, fu = K.fu, V = K.V, s = K.s;
  auto roof = [&](u64 F, u64 B) { return std::fmax((double)F * K.invF, (double)B * K.invB); };
  double tQKV = 0.0, tATTP = 0.0, tATTD = 0.0, tO = 0.0, tUP = 0.0, tDOWN = 0.0, tLM = 0.0;
  if (N > 0) {
    tQKV = roof(2 * N * h * (q + 2 * g), s * (h * (q + 2 * g) + N * h + N * (q + 2 * g)));
    tO = roof(2 * N * q * h, s * (q * h + N * q + N * h));
    tUP = roof(2 * N * h * fu, s * (h * fu + N * h + N * fu));
    tDOWN = roof(2 * N * f * h, s * (f * h + N * f + N * h));
  }
  if (Np > 0) tATTP = roof(4 * q * Ap, s * (Np * (2 * q + 2 * g) + 2 * g * Kp));
  if (D > 0) tATTD = roof(4 * q * Cd, s * (D * (2 * q + 2 * g) + 2 * g * Cd));
  if (S > 0) tLM = roof(2 * S * h * V, s * (V * h + S * h + S * V));
  const double t_layer = ((((tQKV + tATTP) + tATTD) + tO) + tUP) + tDOWN;
  // PRELOAD (reading R-N4): the swap-in streams layer by layer (chunk = swap_in / L bytes, exact
  // since kvb has a factor L) through the buffer while the layers compute; the swap-out before
  // it stays serial.  SEQUENTIAL (A10): every swap byte, then the compute.
  const bool pipe = K.link_mode == OR_LINK_PRELOAD && swap_in > 0;
  double T;
  if (pipe) {
    const u64 chunk = swap_in / K.L;
    const u64 slots = std::max<u64>(1, K.preload_buf / chunk);
    T = pipeline(K.L, (double)chunk * K.invH, t_layer, slots);
  } else {
    T = t_layer * (double)K.L;
  }
  T = T + tLM;
  if (K.tp > 1) {
    const u64 b_ar = 2 * (u64)(K.tp - 1) * N * h * s;
    const double ar = (double)b_ar * K.invT;
    T = T + ar * (double)(2 * K.L);
  }
  const u64 swap_bytes = pipe ? swap_out : swap_out + swap_in;
  if (swap_bytes > 0) {
    const double sw = (double)swap_bytes * K.invH;
    T = T + sw;
  }
  if (fetch_blocks > 0) T = T + (double)fetch_blocks * fetch_s;  // NEXT-2 cache hits
  T = T + K.overhead;
  const double Tn = T * 1e9;
  return (i64)std::floor(Tn + 0.5);
}

struct CostK_ {
  CostCtx k;
};

// ----------------------------------------------------------------- state
enum Kind { K_DEC = 0, K_PRE_FRESH = 1, K_PRE_RECOMP = 2 };

struct Req {
  i64 a = 0;
  u32 p = 0, o = 0;
  u32 status = 0;  // 0 unfinished, 1 finished, 2 rejected
  u64 ctx = 0, gen = 0;
  i64 first_tok = 0, last_tok = 0, max_gap = 0;
  u32 n_preempt = 0;
  std::vector<u32> blocks;  // logical order
  bool pref = false;        // CHUNKED: prefill in progress (blocks held for p + gen)
  u64 pdone = 0;            // CHUNKED: prefill tokens computed so far
  i64 finish = 0;
  u64 finish_k = 0;
};

}  // namespace

struct oracle_run {
  oracle_summary summary;
  std::vector<oracle_record> records;
  std::vector<oracle_iter> iters;
  std::vector<oracle_sample> trace[OR_MAX_WORKERS];
  std::vector<oracle_event> events;
};

namespace {

// ----------------------------------------------------------------- c.6 metrics
void metrics(const oracle_cfg &c, const oracle_derived &d, const std::vector<Req> &req,
             oracle_summary &S) {
  const u64 n = req.size();
  std::vector<double> vals[5];
  double tp_sum = 0.0, norm_sum = 0.0;
  i64 ttft_sum = 0, e2e_sum = 0, mt_sum = 0;
  u64 n_fin = 0, good_mt = 0, good_both = 0;
  i64 last_finish = 0;
  for (u64 i = 0; i < n; ++i) {
    const Req &r = req[i];
    if (r.status != 1) continue;
    const i64 ttft = r.first_tok - r.a, e2e = r.finish - r.a, mt = r.max_gap;
    ++n_fin;
    last_finish = std::max(last_finish, r.finish);
    vals[0].push_back((double)ttft / 1e9);
    vals[2].push_back((double)e2e / 1e9);
    vals[4].push_back((double)mt / 1e9);
    ttft_sum += ttft;
    e2e_sum += e2e;
    mt_sum += mt;
    if (r.o >= 2) {
      const double v = (double)(e2e - ttft) / (double)(r.o - 1);
      vals[1].push_back(v / 1e9);
      tp_sum += v;
    }
    const double nv = (double)e2e / (double)r.o;
    vals[3].push_back(nv / 1e9);
    norm_sum += nv;
    if (mt <= d.slo_mtpot_ns) {
      ++good_mt;
      if (ttft <= d.slo_ttft_ns) ++good_both;
    }
  }
  const u32 qbp[4] = {5000, 9000, 9900, 10000};
  for (int m = 0; m < 5; ++m) {
    std::vector<double> v = vals[m];
    std::sort(v.begin(), v.end());
    const u64 cnt = v.size();
    for (int qi = 0; qi < 4; ++qi) {
      if (cnt == 0) {
        S.stat[m][qi] = 0.0;
        continue;
      }
      u64 rank = ((u64)qbp[qi] * cnt + 9999) / 10000;
      if (rank < 1) rank = 1;
      S.stat[m][qi] = v[rank - 1];
    }
    double mean = 0.0;
    if (cnt > 0) {
      if (m == 0) mean = ((double)ttft_sum / (double)cnt) / 1e9;
      if (m == 2) mean = ((double)e2e_sum / (double)cnt) / 1e9;
      if (m == 4) mean = ((double)mt_sum / (double)cnt) / 1e9;
      if (m == 1) mean = (tp_sum / (double)cnt) / 1e9;
      if (m == 3) mean = (norm_sum / (double)cnt) / 1e9;
    }
    S.stat[m][4] = mean;
  }
  S.last_finish_ns = last_finish;
  S.first_arrival_ns = n ? req[0].a : 0;
  const i64 span = last_finish - S.first_arrival_ns;
  if (n_fin > 0 && span > 0) {
    const double sec = (double)span / 1e9;
    S.throughput_rps = (double)n_fin / sec;
    S.goodput_mtpot_rps = (double)good_mt / sec;
    S.goodput_both_rps = (double)good_both / sec;
  }
  (void)c;
}

// memory trace from the iteration list (c.6 "Memory trace")
void build_trace(const oracle_cfg &c, const std::vector<oracle_iter> &it, u32 worker, i64 t_final,
                 std::vector<oracle_sample> &out, bool &overflow) {
  out.clear();
  if (c.trace_mode == OR_TRACE_FULL) {
    for (const oracle_iter &x : it) {
      if (x.worker != worker) continue;
      if (out.size() >= c.trace_cap_samples) {
        overflow = true;
        break;
      }
      out.push_back({x.t_start, x.T_ns, (u64)x.blocks * (u64)x.T_ns, (u32)x.blocks, 1u});
    }
  } else if (c.trace_mode == OR_TRACE_BINNED) {
    // bins [bW, (b+1)W) for b < ceil(t_final / W); each iteration adds blocks x overlap to every
    // bin it overlaps, and counts in the bin holding its start (reading R5)
    const i64 W = (i64)c.trace_bin_ns;
    const i64 nbins = (t_final + W - 1) / W;
    std::vector<oracle_sample> bins((size_t)nbins);
    for (i64 b = 0; b < nbins; ++b) bins[(size_t)b] = {b * W, W, 0, 0, 0};
    for (const oracle_iter &x : it) {
      if (x.worker != worker) continue;
      const i64 ts = x.t_start, te = x.t_start + x.T_ns;
      const i64 b0 = ts / W;
      if (b0 < nbins) bins[(size_t)b0].n_iter += 1;
      for (i64 b = b0; b < nbins && b * W < te; ++b) {
        const i64 lo = std::max(ts, b * W), hi = std::min(te, (b + 1) * W);
        if (hi - lo > 0) {
          bins[(size_t)b].block_ns += x.blocks * (u64)(hi - lo);
          bins[(size_t)b].blocks_max = std::max<u32>(bins[(size_t)b].blocks_max, (u32)x.blocks);
        }
      }
    }
    if ((u64)nbins > c.trace_cap_samples) {
      overflow = true;
      bins.resize((size_t)c.trace_cap_samples);
    }
    out = bins;
  }
}

bool check_invariants(const std::vector<Req> &req, const std::set<u32> &R, const std::set<u32> &Q,
                      const std::set<u32> &freeset, u64 total, u64 bs) {
  std::set<u32> seen(freeset.begin(), freeset.end());
  u64 alloc = 0;
  u32 n_pref = 0;
  for (u32 id : R) {
    const Req &r = req[id];
    // a chunked prefill in progress holds the blocks of its whole target p + gen (reading R-N3b)
    const u64 want = r.pref ? ceil_div((u64)r.p + r.gen, bs) : ceil_div(r.ctx, bs);
    if (r.blocks.size() != want) return fail("held != ceil(ctx/bs) for request " + std::to_string(id));
    if (r.pref) {
      // derived property of R-N3b (the budget runs out at the last prefill entry): at most one
      // prefill is in progress and it is the latest arrival in R
      if (++n_pref > 1 || id != *R.rbegin()) return fail("chunked prefill not at the tail of R");
      if (r.pdone == 0 || r.pdone >= (u64)r.p + r.gen) return fail("chunk progress out of range");
    }
    for (u32 b : r.blocks) {
      if (b >= total) return fail("block id out of range");
      if (!seen.insert(b).second) return fail("block " + std::to_string(b) + " in two lists");
      ++alloc;
    }
  }
  for (u32 id : Q) {
    if (!req[id].blocks.empty()) return fail("queued request holds blocks");
    if (R.count(id)) return fail("request in both R and Q");
  }
  if (freeset.size() + alloc != total) return fail("free + allocated != total");
  return true;
}

// ----------------------------------------------------------------- c.4 unified worker loop
oracle_run *simulate_unified(const oracle_cfg &c) {
  oracle_derived d;
  if (!derive(c, 0, d)) return nullptr;
  if (c.iter_mode == OR_CHUNKED && c.max_batched_tokens < c.max_num_seqs) {
    g_err = "CHUNKED needs max_batched_tokens >= max_num_seqs (every decode fits the budget)";
    return nullptr;
  }
  const CostCtx K = cost_ctx(c, d, 0);
  std::vector<i64> A;
  std::vector<u32> Pl, Ol;
  if (!workload(c, A, Pl, Ol)) return nullptr;
  const u32 n = c.num_requests;
  const u64 bs = c.block_size, total = d.total_blocks;
  const bool SWAPM = c.preempt == OR_SWAP;
  const bool RATIO = c.kind == OR_CONT_RATIO;

  std::vector<Req> req(n);
  for (u32 i = 0; i < n; ++i) {
    req[i].a = A[i];
    req[i].p = Pl[i];
    req[i].o = Ol[i];
  }
  oracle_run *run = new oracle_run();
  std::memset(&run->summary, 0, sizeof(run->summary));
  oracle_summary &S = run->summary;

  std::set<u32> freeset;
  for (u64 b = 0; b < total; ++b) freeset.insert((u32)b);
  std::set<u32> R, Q;
  i64 t = 0;
  u64 k = 0;
  u32 arr = 0, adm = 0;
  u64 sched_d = 0, block_d = 0, req_d = 0;
  u64 req_iters = 0, n_preempt_total = 0, swap_out_total = 0, swap_in_total = 0;
  u64 peak = 0, block_ns_sum = 0, n_rej_total = 0;

  auto alloc_lowest = [&](u32 id, u64 cnt) {
    for (u64 j = 0; j < cnt; ++j) {
      const u32 b = *freeset.begin();
      freeset.erase(freeset.begin());
      req[id].blocks.push_back(b);
      block_d += fold_block(k, 1, id, b);
      if (c.keep_events) run->events.push_back({k, 1, id, b, 0});
    }
  };
  auto free_all = [&](u32 id) {
    for (u32 b : req[id].blocks) {  // logical order
      freeset.insert(b);
      block_d += fold_block(k, 2, id, b);
      if (c.keep_events) run->events.push_back({k, 2, id, b, 0});
    }
    req[id].blocks.clear();
  };

  while (true) {
    // 0. termination
    if (adm == n && R.empty() && Q.empty()) break;
    if (c.horizon_ns >= 0 && t >= c.horizon_ns) {
      S.status_flags |= 4;
      break;
    }
    // 1. ingest: requests with a_i <= t are visible at this boundary (reading A2)
    while (arr < n && req[arr].a <= t) ++arr;
    // 2. idle skip
    if (R.empty() && Q.empty() && adm == arr) {
      t = req[arr].a;
      continue;
    }
    std::map<u32, Kind> kind;  // this iteration's batch: id -> entry kind
    u64 n_res = 0, n_adm = 0, n_rej = 0, swap_in = 0, m = 0, swap_out = 0;
    // NEXT-3 prefill-first (vLLM v0.6.2 default, reading R-N3): when fresh requests can be
    // admitted the iteration runs only their prefills; the running requests pause
    const bool CH = c.iter_mode == OR_CHUNKED;
    std::map<u32, u64> chunk;  // CHUNKED: this iteration's chunk length per prefill entry
    auto fresh_admission = [&](u64 tokens) {
      while (adm < arr) {
        Req &x = req[adm];
        const u64 need = ceil_div(x.p, bs);
        const u64 cap = RATIO ? d.ratio_limit : total - c.watermark_blocks;
        if (need > cap) {
          x.status = 2;
          ++n_rej;
          ++adm;
          continue;
        }
        const u64 fr = freeset.size();
        if (R.size() + 1 > c.max_num_seqs) break;
        // CHUNKED (R-N3b): one token of budget suffices; the chunk is what is left of it
        if (CH ? tokens + 1 > c.max_batched_tokens : tokens + x.p > c.max_batched_tokens) break;
        if ((i64)fr - (i64)need < (i64)c.watermark_blocks) break;
        if (RATIO && (total - fr) + need > d.ratio_limit) break;
        alloc_lowest(adm, need);
        R.insert(adm);
        kind[adm] = K_PRE_FRESH;
        if (CH) {
          const u64 ch = std::min<u64>(x.p, c.max_batched_tokens - tokens);
          x.pref = true;
          x.pdone = 0;
          chunk[adm] = ch;
          tokens += ch;
        } else {
          tokens += x.p;
        }
        ++n_adm;
        ++adm;
      }
    };
    const bool PF = c.iter_mode == OR_PREFILL_FIRST;
    if (PF && Q.empty() && (c.kind != OR_STATIC || R.empty())) fresh_admission(0);
    const bool pf_only = PF && n_adm > 0;
    // 3. decode reservation + preemption (reading A7)
    const u64 F = freeset.size();
    std::vector<u32> Rv;
    if (!pf_only) Rv.assign(R.begin(), R.end());
    // a prefill in progress decodes nothing and already holds its blocks (R-N3b)
    auto need_of = [&](u32 id) -> u64 { return (!req[id].pref && req[id].ctx % bs == 0) ? 1 : 0; };
    u64 sum_need = 0;
    for (u32 id : Rv) sum_need += need_of(id);
    if (sum_need > F) {
      const u64 nr = Rv.size();
      for (m = 1; m <= nr; ++m) {
        u64 lhs = 0, rhs = F;
        for (u64 j = 0; j < nr - m; ++j) lhs += need_of(Rv[j]);
        for (u64 j = nr - m; j < nr; ++j) rhs += req[Rv[j]].blocks.size();
        if (lhs <= rhs) break;
      }
      if (m >= nr) {
        g_err = "preemption would evict r_1 (validation should make this impossible)";
        delete run;
        return nullptr;
      }
      for (u64 i = 0; i < m; ++i) {  // r_n, r_{n-1}, ..., r_{n-m+1}
        const u32 id = Rv[nr - 1 - i];
        Req &x = req[id];
        const u64 held = x.blocks.size();
        free_all(id);
        x.n_preempt += 1;
        if (x.pref) {  // partial prefill: its KV is discarded whatever the mode (R-N3b)
          x.pref = false;
          x.pdone = 0;
          x.ctx = 0;
        } else if (SWAPM) {
          swap_out += held * d.block_bytes;
        } else {
          x.ctx = 0;
        }
        R.erase(id);
        Q.insert(id);
      }
      n_preempt_total += m;
    }
    u64 D3 = 0;
    if (!pf_only) {
      for (u32 id : R) {  // surviving requests, ascending id
        if (req[id].pref) continue;
        kind[id] = K_DEC;
        ++D3;
        if (need_of(id)) alloc_lowest(id, 1);
      }
    }
    u64 tokens = D3;
    if (CH) {
      // continuing chunked prefills take the budget left by the decodes, in id order (R-N3b)
      for (u32 id : R) {
        Req &x = req[id];
        if (!x.pref) continue;
        const u64 ch = std::min<u64>((u64)x.p + x.gen - x.pdone, c.max_batched_tokens - tokens);
        if (ch == 0) continue;  // no budget left: it sits this iteration out
        kind[id] = x.gen == 0 ? K_PRE_FRESH : K_PRE_RECOMP;
        chunk[id] = ch;
        tokens += ch;
      }
    }
    if (m == 0 && !pf_only) {
      // 4. resume, head first, stop at the first misfit (reading A6)
      std::vector<u32> Qv(Q.begin(), Q.end());
      for (u32 id : Qv) {
        Req &x = req[id];
        u64 need, tok;
        // re-prefill p + gen under RECOMPUTE, and (CHUNKED) after losing a partial prefill
        const bool recomp = !SWAPM || x.ctx == 0;
        if (!recomp) {
          need = ceil_div(x.ctx, bs) + ((x.ctx % bs == 0) ? 1 : 0);
          tok = 1;
        } else {
          need = ceil_div(x.p + x.gen, bs);
          tok = x.p + x.gen;
        }
        const bool ok = (R.size() + 1 <= c.max_num_seqs) &&
                        (CH ? tokens + 1 <= c.max_batched_tokens : tokens + tok <= c.max_batched_tokens) &&
                        ((i64)freeset.size() - (i64)need >= (i64)c.watermark_blocks);
        if (!ok) break;
        alloc_lowest(id, need);
        Q.erase(id);
        R.insert(id);
        ++n_res;
        if (CH && recomp) {
          const u64 ch = std::min<u64>(tok, c.max_batched_tokens - tokens);
          x.pref = true;
          x.pdone = 0;
          chunk[id] = ch;
          tokens += ch;
        } else {
          tokens += tok;
        }
        if (!recomp) {
          swap_in += ceil_div(x.ctx, bs) * d.block_bytes;
          kind[id] = K_DEC;
        } else {
          // gen = 0: a chunked prefill lost before its first token starts over as a fresh one
          kind[id] = x.gen == 0 ? K_PRE_FRESH : K_PRE_RECOMP;
        }
      }
      // 5. fresh FCFS admission (STATIC P:167/A16; ratio P:460/A15); in
      // prefill-first mode it was already attempted at the top of the pass
      if (!PF && Q.empty() && (c.kind != OR_STATIC || R.empty())) fresh_admission(tokens);
    }
    n_rej_total += n_rej;
    // 6. empty batch
    if (kind.empty()) continue;
    // 7. cost (c.5)
    std::vector<Prefill> pf;
    std::vector<u64> dec;
    u64 Np = 0, Cd = 0;
    for (const auto &kv : kind) {
      const u32 id = kv.first;
      const Req &x = req[id];
      if (kv.second == K_DEC) {
        dec.push_back(x.ctx + 1);
        Cd += x.ctx + 1;
      } else if (CH) {  // a chunk of L tokens after pdone computed ones (R-N3b)
        const u64 L = chunk.at(id);
        pf.push_back({L, x.pdone, x.pdone + L == (u64)x.p + x.gen});
        Np += L;
      } else if (kv.second == K_PRE_FRESH) {
        pf.push_back({x.p, 0});
        Np += x.p;
      } else {
        pf.push_back({x.p + x.gen, 0});
        Np += x.p + x.gen;
      }
    }
    const i64 T = iter_time(K, pf, dec, swap_out, swap_in);
    // 8. commit
    const i64 ts = t, te = t + T;
    const u64 blocks = total - freeset.size();
    const u64 entries = kind.size();
    u64 n_fin = 0;
    for (const auto &kv : kind) {
      const u32 id = kv.first;
      Req &x = req[id];
      const Kind kd = kv.second;
      if (CH && kd != K_DEC) {
        x.pdone += chunk.at(id);
        if (x.pdone < (u64)x.p + x.gen) continue;  // non-final chunk: no token yet
        x.pref = false;
        x.pdone = 0;
      }
      if (kd == K_PRE_FRESH) {
        x.ctx = x.p;
        x.gen = 1;
        x.first_tok = te;
        x.last_tok = te;
      } else {
        if (kd == K_PRE_RECOMP) {
          x.ctx = x.p + x.gen;
          x.gen += 1;
        } else {
          x.ctx += 1;
          x.gen += 1;
        }
        const i64 gap = te - x.last_tok;
        x.max_gap = std::max(x.max_gap, gap);
        x.last_tok = te;
      }
      if (x.gen == x.o) {
        x.status = 1;
        x.finish = te;
        x.finish_k = k;
        req_d += fold({id, (u64)(x.first_tok - x.a), (u64)(x.finish - x.a), (u64)x.max_gap,
                       x.n_preempt, k});
        free_all(id);
        R.erase(id);
        ++n_fin;
      }
    }
    sched_d += fold_sched(k, (u64)ts, (u64)T, pf.size(), dec.size(), Np, Cd, m, n_res, n_adm, n_rej,
                     n_fin, blocks);
    run->iters.push_back({k, ts, T, pf.size(), dec.size(), Np, Cd, m, n_res, n_adm, n_rej, n_fin,
                          blocks, 0, 0});
    req_iters += entries;
    peak = std::max(peak, blocks);
    block_ns_sum += blocks * (u64)T;
    swap_out_total += swap_out;
    swap_in_total += swap_in;
    if (te < t) {
      g_err = "clock went backwards";
      delete run;
      return nullptr;
    }
    t = te;
    ++k;
    if (c.check_invariants && !check_invariants(req, R, Q, freeset, total, bs)) {
      delete run;
      return nullptr;
    }
  }

  // records + summary
  run->records.resize(n);
  u64 n_fin = 0;
  for (u32 i = 0; i < n; ++i) {
    const Req &x = req[i];
    oracle_record &rec = run->records[i];
    rec.ttft_ns = (x.gen >= 1 || x.status == 1) ? x.first_tok - x.a : 0;
    rec.e2e_ns = x.status == 1 ? x.finish - x.a : 0;
    rec.mtpot_ns = x.status == 1 ? x.max_gap : 0;
    rec.n_preempt = x.n_preempt;
    rec.status = x.status;
    rec.finish_k = x.status == 1 ? x.finish_k : 0;
    if (x.status == 1) ++n_fin;
  }
  S.n_requests = n;
  S.n_finished = n_fin;
  S.n_rejected = n_rej_total;
  S.n_unfinished = n - n_fin - n_rej_total;
  if (n_rej_total == n) S.status_flags |= 2;
  S.n_iterations = k;
  S.n_request_iterations = req_iters;
  S.n_preemptions = n_preempt_total;
  S.swap_out_bytes = swap_out_total;
  S.swap_in_bytes = swap_in_total;
  S.t_final = t;
  S.sched_digest = sched_d;
  S.block_digest = block_d;
  S.request_digest = req_d;
  S.total_blocks = total;
  S.peak_blocks = peak;
  S.block_ns_sum = block_ns_sum;
  S.mean_util = (t > 0 && total > 0) ? (double)block_ns_sum / ((double)total * (double)t) : 0.0;
  metrics(c, d, req, S);
  bool ovf = false;
  build_trace(c, run->iters, 0, t, run->trace[0], ovf);
  if (ovf) S.status_flags |= 1;
  return run;
}

// ----------------------------------------------------------------- a.9 P/D pair
// SURVEY §8(a.9), readings A35 and R-PD1..R-PD7 in DESIGN.md.  Two workers per point: P runs
// prefill-only iterations and emits the first token; at the end-of-prefill
// breakpoint the request joins D's pending FIFO still holding its P blocks; D pulls pending
// requests FCFS at its boundaries, allocates ceil(p/bs) blocks and starts a p*kvb-byte transfer on
// the FIFO P->D link; the request becomes runnable on D at the first D boundary
// >= transfer end; P frees its blocks at its first boundary >= transfer end.  The two workers are
// advanced in time order of their next boundary, D first on ties (reading A2).  An idle worker
// wakes at the earliest event that can change its decision.
oracle_run *simulate_pd(const oracle_cfg &c) {
  if (c.kind == OR_CONT_RATIO || c.iter_mode != OR_MIXED) {
    g_err = "PD_PAIR supports STATIC and CONT policies in MIXED mode only";
    return nullptr;
  }
  oracle_derived dP, dD;
  if (!derive(c, 0, dP) || !derive(c, 1, dD)) return nullptr;
  const CostK_ KP = {cost_ctx(c, dP, 0)}, KD = {cost_ctx(c, dD, 1)};
  std::vector<i64> A;
  std::vector<u32> Pl, Ol;
  if (!workload(c, A, Pl, Ol)) return nullptr;
  const u32 n = c.num_requests;
  const u64 bs = c.block_size, totP = dP.total_blocks, totD = dD.total_blocks;
  const bool SWAPM = c.preempt == OR_SWAP;
  const i64 INF = INT64_MAX;
  const double inv_link = 1.0 / c.pd_link_bw;

  struct PReq {
    i64 a = 0;
    u32 p = 0, o = 0, status = 0;
    u64 ctx = 0, gen = 0;
    i64 first_tok = 0, last_tok = 0, max_gap = 0, finish = 0, join = 0, xend = 0;
    u32 n_preempt = 0;
    bool xstarted = false;
    std::vector<u32> pblocks, dblocks;
    u64 finish_k = 0;
  };
  std::vector<PReq> req(n);
  for (u32 i = 0; i < n; ++i) {
    req[i].a = A[i];
    req[i].p = Pl[i];
    req[i].o = Ol[i];
  }
  oracle_run *run = new oracle_run();
  std::memset(&run->summary, 0, sizeof(run->summary));
  oracle_summary &S = run->summary;
  std::set<u32> freeP, freeD;
  for (u64 b = 0; b < totP; ++b) freeP.insert((u32)b);
  for (u64 b = 0; b < totD; ++b) freeD.insert((u32)b);
  std::deque<u32> pending;    // finished prefill, waiting for D admission (join order = id order)
  std::deque<u32> pholders;   // hold P blocks until their transfer ends (same FIFO order)
  std::set<u32> xfer, R, Q;   // D: transferring, running, preempted
  i64 tP = 0, tD = 0, link_busy = 0, lastP = 0, lastD = 0;
  bool P_idle = false, D_idle = false;
  u64 kP = 0, kD = 0;
  u32 arr = 0, adm = 0, n_done = 0;
  u64 sched_d = 0, block_d = 0, req_d = 0, req_iters = 0, npre = 0, swo = 0, swi = 0, nrej_tot = 0;
  u64 peakD = 0, bnsD = 0, n_xfer = 0, xfer_bytes = 0;

  auto ev = [&](u64 k, u32 kind, u32 worker, u32 id, u32 b) {
    block_d += fold_block(k, kind + 2 * worker, id, b);
    if (c.keep_events) run->events.push_back({k, kind, id, b, worker});
  };
  auto finish_req = [&](u32 id, i64 te, u64 k) {
    PReq &x = req[id];
    x.status = 1;
    x.finish = te;
    x.finish_k = k;
    req_d += fold({id, (u64)(x.first_tok - x.a), (u64)(x.finish - x.a), (u64)x.max_gap, x.n_preempt, k});
    ++n_done;
  };

  while (true) {
    if (n_done == n) break;
    const i64 tnext = std::min(tP, tD);
    if (tnext == INF) {
      g_err = "P/D deadlock: both workers wait";
      delete run;
      return nullptr;
    }
    if (c.horizon_ns >= 0 && tnext >= c.horizon_ns) {
      S.status_flags |= 4;
      break;
    }
    if (tD <= tP) {
      // ================================================================ D boundary
      const i64 t = tD;
      // 1. finished transfers become runnable (ascending id)
      std::vector<u32> xv(xfer.begin(), xfer.end());
      for (u32 id : xv) {
        if (req[id].xend <= t) {
          xfer.erase(id);
          R.insert(id);
        }
      }
      std::map<u32, Kind> kind;
      // 3. decode reservation + preemption over R
      const u64 F = freeD.size();
      std::vector<u32> Rv(R.begin(), R.end());
      auto need_of = [&](u32 id) -> u64 { return (req[id].ctx % bs == 0) ? 1 : 0; };
      u64 sum_need = 0;
      for (u32 id : Rv) sum_need += need_of(id);
      u64 m = 0, swap_out = 0;
      if (sum_need > F) {
        const u64 nr = Rv.size();
        for (m = 1; m <= nr; ++m) {
          u64 lhs = 0, rhs = F;
          for (u64 j = 0; j < nr - m; ++j) lhs += need_of(Rv[j]);
          for (u64 j = nr - m; j < nr; ++j) rhs += req[Rv[j]].dblocks.size();
          if (lhs <= rhs) break;
        }
        // blocks held by in-flight transfers are not preemptible, so on D the minimal m may
        // be all of R (reading R-PD4); m <= nr always holds since m = nr satisfies the condition
        if (m > nr) {
          g_err = "P/D: no victim count satisfies c.4 step 3";
          delete run;
          return nullptr;
        }
        for (u64 i = 0; i < m; ++i) {
          const u32 id = Rv[nr - 1 - i];
          PReq &x = req[id];
          const u64 held = x.dblocks.size();
          for (u32 b : x.dblocks) {
            freeD.insert(b);
            ev(kD, 2, 1, id, b);
          }
          x.dblocks.clear();
          x.n_preempt += 1;
          if (SWAPM) swap_out += held * dD.block_bytes;
          else x.ctx = 0;
          R.erase(id);
          Q.insert(id);
        }
        npre += m;
      }
      for (u32 id : R) {
        kind[id] = K_DEC;
        if (need_of(id)) {
          const u32 b = *freeD.begin();
          freeD.erase(freeD.begin());
          req[id].dblocks.push_back(b);
          ev(kD, 1, 1, id, b);
        }
      }
      const u64 D3 = R.size();
      u64 n_res = 0, n_adm = 0, swap_in = 0, tokens = D3;
      if (m == 0) {
        // 4. resume (|R| counts transferring requests too)
        std::vector<u32> Qv(Q.begin(), Q.end());
        for (u32 id : Qv) {
          PReq &x = req[id];
          u64 need, tok;
          if (SWAPM) {
            need = ceil_div(x.ctx, bs) + ((x.ctx % bs == 0) ? 1 : 0);
            tok = 1;
          } else {
            need = ceil_div(x.p + x.gen, bs);
            tok = x.p + x.gen;
          }
          const bool ok = (R.size() + xfer.size() + 1 <= c.max_num_seqs) &&
                          (tokens + tok <= c.max_batched_tokens) &&
                          ((i64)freeD.size() - (i64)need >= (i64)c.watermark_blocks);
          if (!ok) break;
          for (u64 j = 0; j < need; ++j) {
            const u32 b = *freeD.begin();
            freeD.erase(freeD.begin());
            x.dblocks.push_back(b);
            ev(kD, 1, 1, id, b);
          }
          Q.erase(id);
          R.insert(id);
          ++n_res;
          tokens += tok;
          if (SWAPM) {
            swap_in += ceil_div(x.ctx, bs) * dD.block_bytes;
            kind[id] = K_DEC;
          } else {
            kind[id] = K_PRE_RECOMP;
          }
        }
        // 5. pull pending requests (FCFS), start their KV transfers
        if (Q.empty() && (c.kind != OR_STATIC || (R.empty() && xfer.empty()))) {
          while (!pending.empty() && req[pending.front()].join <= t) {
            const u32 id = pending.front();
            PReq &x = req[id];
            const u64 need = ceil_div(x.p, bs);
            if (R.size() + xfer.size() + 1 > c.max_num_seqs) break;
            if ((i64)freeD.size() - (i64)need < (i64)c.watermark_blocks) break;
            for (u64 j = 0; j < need; ++j) {
              const u32 b = *freeD.begin();
              freeD.erase(freeD.begin());
              x.dblocks.push_back(b);
              ev(kD, 1, 1, id, b);
            }
            const u64 bytes = (u64)x.p * dD.kvb;
            const double sec = (double)bytes * inv_link;
            const i64 dur = (i64)std::floor(sec * 1e9 + 0.5);
            const i64 start = std::max(t, link_busy);
            x.xend = start + dur;
            x.xstarted = true;
            link_busy = x.xend;
            xfer.insert(id);
            pending.pop_front();
            ++n_adm;
            ++n_xfer;
            xfer_bytes += bytes;
            if (P_idle && x.xend < tP) tP = x.xend;  // P may be waiting for these P blocks
          }
        }
      }
      if (R.empty()) {  // 6. nothing runnable: wait for a transfer end or a pending join
        i64 wake = INF;
        for (u32 id : xfer) wake = std::min(wake, req[id].xend);
        for (u32 id : pending)
          if (req[id].join > t) wake = std::min(wake, req[id].join);
        tD = wake;
        D_idle = true;
        continue;
      }
      // 7. cost on D's profile
      std::vector<Prefill> pf;
      std::vector<u64> dec;
      u64 Np = 0, Cd = 0;
      for (u32 id : R) {
        const PReq &x = req[id];
        if (kind[id] == K_DEC) {
          dec.push_back(x.ctx + 1);
          Cd += x.ctx + 1;
        } else {
          pf.push_back({x.p + x.gen, 0});
          Np += x.p + x.gen;
        }
      }
      const i64 T = iter_time(KD.k, pf, dec, swap_out, swap_in);
      const i64 te = t + T;
      const u64 blocks = totD - freeD.size();
      const u64 entries = R.size();
      u64 n_fin = 0;
      std::vector<u32> Rc(R.begin(), R.end());
      for (u32 id : Rc) {
        PReq &x = req[id];
        if (kind[id] == K_PRE_RECOMP) {
          x.ctx = x.p + x.gen;
          x.gen += 1;
        } else {
          x.ctx += 1;
          x.gen += 1;
        }
        const i64 gap = te - x.last_tok;
        x.max_gap = std::max(x.max_gap, gap);
        x.last_tok = te;
        if (x.gen == x.o) {
          finish_req(id, te, kD);
          for (u32 b : x.dblocks) {
            freeD.insert(b);
            ev(kD, 2, 1, id, b);
          }
          x.dblocks.clear();
          R.erase(id);
          ++n_fin;
        }
      }
      sched_d += fold_sched(kD | (1ull << 40), (u64)t, (u64)T, pf.size(), dec.size(), Np, Cd, m, n_res, n_adm, 0, n_fin,
                       blocks);
      run->iters.push_back({kD, t, T, pf.size(), dec.size(), Np, Cd, m, n_res, n_adm, 0, n_fin, blocks, 1, 0});
      req_iters += entries;
      peakD = std::max(peakD, blocks);
      bnsD += blocks * (u64)T;
      swo += swap_out;
      swi += swap_in;
      tD = te;
      lastD = te;
      ++kD;
      D_idle = false;
    } else {
      // ================================================================ P boundary
      const i64 t = tP;
      // P blocks of finished transfers are freed (transfer order)
      while (!pholders.empty()) {
        const u32 id = pholders.front();
        PReq &x = req[id];
        if (!(x.xstarted && x.xend <= t)) break;
        for (u32 b : x.pblocks) {
          freeP.insert(b);
          ev(kP, 2, 0, id, b);
        }
        x.pblocks.clear();
        pholders.pop_front();
      }
      while (arr < n && req[arr].a <= t) ++arr;
      std::vector<u32> batch;
      u64 tokens = 0, n_rej = 0;
      while (adm < arr) {
        PReq &x = req[adm];
        const u64 need = ceil_div(x.p, bs);
        if (need > totP - c.watermark_blocks) {
          x.status = 2;
          ++n_rej;
          ++n_done;
          ++adm;
          continue;
        }
        if (batch.size() + 1 > c.max_num_seqs) break;
        if (tokens + x.p > c.max_batched_tokens) break;
        if ((i64)freeP.size() - (i64)need < (i64)c.watermark_blocks) break;
        for (u64 j = 0; j < need; ++j) {
          const u32 b = *freeP.begin();
          freeP.erase(freeP.begin());
          x.pblocks.push_back(b);
          ev(kP, 1, 0, adm, b);
        }
        batch.push_back(adm);
        tokens += x.p;
        ++adm;
      }
      nrej_tot += n_rej;
      if (batch.empty()) {  // idle: wait for an arrival or for P blocks to come back
        i64 wake = arr < n ? req[arr].a : INF;
        if (!pholders.empty() && req[pholders.front()].xstarted) wake = std::min(wake, req[pholders.front()].xend);
        tP = wake;
        P_idle = true;
        continue;
      }
      std::vector<Prefill> pf;
      u64 Np = 0;
      for (u32 id : batch) {
        pf.push_back({req[id].p, 0});
        Np += req[id].p;
      }
      const i64 T = iter_time(KP.k, pf, {}, 0);
      const i64 te = t + T;
      const u64 blocks = totP - freeP.size();
      u64 n_fin = 0;
      for (u32 id : batch) {  // the first token; the end-of-prefill breakpoint
        PReq &x = req[id];
        x.ctx = x.p;
        x.gen = 1;
        x.first_tok = te;
        x.last_tok = te;
        if (x.gen == x.o) {
          finish_req(id, te, kP);
          for (u32 b : x.pblocks) {
            freeP.insert(b);
            ev(kP, 2, 0, id, b);
          }
          x.pblocks.clear();
          ++n_fin;
        } else {
          x.join = te;
          pending.push_back(id);
          pholders.push_back(id);
        }
      }
      sched_d += fold_sched(kP, (u64)t, (u64)T, pf.size(), 0, Np, 0, 0, 0, batch.size(), n_rej, n_fin, blocks);
      run->iters.push_back({kP, t, T, pf.size(), 0, Np, 0, 0, 0, batch.size(), n_rej, n_fin, blocks, 0, 0});
      req_iters += batch.size();
      tP = te;
      lastP = te;
      ++kP;
      P_idle = false;
      if (D_idle && te < tD) tD = te;  // new pending requests join at te
    }
    if (c.check_invariants) {
      // conservation on both workers; held = ceil(ctx/bs) on D's running set
      u64 hp = 0, hd = 0;
      for (u32 i = 0; i < n; ++i) {
        hp += req[i].pblocks.size();
        hd += req[i].dblocks.size();
      }
      bool ok = hp + freeP.size() == totP && hd + freeD.size() == totD;
      for (u32 id : R) ok &= req[id].dblocks.size() == ceil_div(req[id].ctx, bs);
      for (u32 id : xfer) ok &= req[id].dblocks.size() == ceil_div(req[id].p, bs);
      for (u32 id : Q) ok &= req[id].dblocks.empty();
      if (!ok) {
        g_err = "P/D invariant violated";
        delete run;
        return nullptr;
      }
    }
  }

  run->records.resize(n);
  u64 n_fin = 0;
  for (u32 i = 0; i < n; ++i) {
    const PReq &x = req[i];
    oracle_record &rec = run->records[i];
    rec.ttft_ns = (x.gen >= 1 || x.status == 1) ? x.first_tok - x.a : 0;
    rec.e2e_ns = x.status == 1 ? x.finish - x.a : 0;
    rec.mtpot_ns = x.status == 1 ? x.max_gap : 0;
    rec.n_preempt = x.n_preempt;
    rec.status = x.status;
    rec.finish_k = x.status == 1 ? x.finish_k : 0;
    if (x.status == 1) ++n_fin;
  }
  const i64 t_final = std::max(lastP, lastD);
  S.n_requests = n;
  S.n_finished = n_fin;
  S.n_rejected = nrej_tot;
  S.n_unfinished = n - n_fin - nrej_tot;
  if (nrej_tot == n) S.status_flags |= 2;
  S.n_iterations = kP + kD;
  S.n_request_iterations = req_iters;
  S.n_preemptions = npre;
  S.swap_out_bytes = swo;
  S.swap_in_bytes = swi;
  S.t_final = t_final;
  S.sched_digest = sched_d;
  S.block_digest = block_d;
  S.request_digest = req_d;
  S.total_blocks = totD;
  S.peak_blocks = peakD;
  S.block_ns_sum = bnsD;
  S.mean_util = (t_final > 0 && totD > 0) ? (double)bnsD / ((double)totD * (double)t_final) : 0.0;
  S.n_transfers = n_xfer;
  S.transfer_bytes = xfer_bytes;
  // metrics over records (same definitions as the unified worker)
  std::vector<Req> rr(n);
  for (u32 i = 0; i < n; ++i) {
    rr[i].a = req[i].a;
    rr[i].p = req[i].p;
    rr[i].o = req[i].o;
    rr[i].status = req[i].status;
    rr[i].first_tok = req[i].first_tok;
    rr[i].finish = req[i].finish;
    rr[i].max_gap = req[i].max_gap;
  }
  metrics(c, dD, rr, S);
  bool ovf = false;
  build_trace(c, run->iters, 0, t_final, run->trace[0], ovf);
  build_trace(c, run->iters, 1, t_final, run->trace[1], ovf);
  if (ovf) S.status_flags |= 1;
  return run;
}

// ----------------------------------------------------------------- NEXT-1 xP:yD node
// SURVEY §8(f) NEXT-1 and readings R-X1..R-X6 in DESIGN.md.  x prefill workers P_0..P_{x-1} (the
// prefill profile) and y decode workers D_0..D_{y-1} (the decode profile) run the a.9 worker
// loops; a global scheduler dispatches every arrival to a prefill
// worker and, at the end-of-prefill breakpoint, every request to a decode worker.  Dispatch
// events at time t are handled before worker boundaries at t (reading A2), in request-id order;
// boundaries at equal times go decode workers first, then prefill workers, lower index first.
// Each decode worker has its own FIFO ingress link.  With x = y = 1 this is exactly simulate_pd.
oracle_run *simulate_pdn(const oracle_cfg &c) {
  const u32 X = c.n_prefill ? c.n_prefill : 1, Y = c.n_decode ? c.n_decode : 1;
  if (c.kind == OR_CONT_RATIO || c.iter_mode != OR_MIXED) {
    g_err = "PD_PAIR supports STATIC and CONT policies in MIXED mode only";
    return nullptr;
  }
  if (X + Y > OR_MAX_WORKERS || c.dispatch > OR_DISPATCH_LEAST_MEMORY) {
    g_err = "PD node: need x + y <= 8 workers and a known dispatch policy";
    return nullptr;
  }
  oracle_derived dP, dD;
  if (!derive(c, 0, dP) || !derive(c, 1, dD)) return nullptr;
  const CostK_ KP = {cost_ctx(c, dP, 0)}, KD = {cost_ctx(c, dD, 1)};
  std::vector<i64> A;
  std::vector<u32> Pl, Ol;
  if (!workload(c, A, Pl, Ol)) return nullptr;
  const u32 n = c.num_requests;
  const u64 bs = c.block_size, totP = dP.total_blocks, totD = dD.total_blocks;
  const bool SWAPM = c.preempt == OR_SWAP;
  const i64 INF = INT64_MAX;
  const double inv_link = 1.0 / c.pd_link_bw;

  struct NReq {
    i64 a = 0;
    u32 p = 0, o = 0, status = 0;
    u64 ctx = 0, gen = 0;
    i64 first_tok = 0, last_tok = 0, max_gap = 0, finish = 0, join = 0, xend = 0;
    u32 n_preempt = 0, pw = 0, dw = 0;
    bool xstarted = false;
    std::vector<u32> pblocks, dblocks;
    u64 finish_k = 0;
  };
  struct PW {  // a prefill worker
    std::set<u32> free;
    std::deque<u32> queue;      // dispatched, not yet admitted (dispatch order)
    std::vector<u32> batch;     // the running prefill batch, dispatched onward at tdisp
    std::set<u32> holders;      // finished prefill, P blocks held until the transfer ends
    i64 t = 0, tdisp = INT64_MAX, last = 0;
    u64 k = 0;
    bool idle = false;
  };
  struct DW {  // a decode worker
    std::set<u32> free;
    std::deque<u32> pending;    // dispatched, not yet pulled (dispatch order)
    std::set<u32> xfer, R, Q;
    i64 t = 0, link_busy = 0, last = 0;
    u64 k = 0, peak = 0, bns = 0;
    bool idle = false;
  };
  std::vector<NReq> req(n);
  for (u32 i = 0; i < n; ++i) {
    req[i].a = A[i];
    req[i].p = Pl[i];
    req[i].o = Ol[i];
  }
  std::vector<PW> Pw(X);
  std::vector<DW> Dw(Y);
  for (PW &w : Pw)
    for (u64 b = 0; b < totP; ++b) w.free.insert((u32)b);
  for (DW &w : Dw)
    for (u64 b = 0; b < totD; ++b) w.free.insert((u32)b);
  oracle_run *run = new oracle_run();
  std::memset(&run->summary, 0, sizeof(run->summary));
  oracle_summary &S = run->summary;
  u32 arr = 0, n_done = 0;
  u64 rrP = 0, rrD = 0;
  u64 sched_d = 0, block_d = 0, req_d = 0, req_iters = 0, npre = 0, swo = 0, swi = 0, nrej_tot = 0;
  u64 n_xfer = 0, xfer_bytes = 0;

  auto ev = [&](u64 k, u32 kind, u32 worker, u32 id, u32 b) {
    block_d += fold_block(k, kind + 2 * worker, id, b);
    if (c.keep_events) run->events.push_back({k, kind, id, b, worker});
  };
  auto finish_req = [&](u32 id, i64 te, u64 k) {
    NReq &x = req[id];
    x.status = 1;
    x.finish = te;
    x.finish_k = k;
    req_d += fold({id, (u64)(x.first_tok - x.a), (u64)(x.finish - x.a), (u64)x.max_gap, x.n_preempt, k});
    ++n_done;
  };
  // the global scheduler (reading R-X2): round robin in dispatch order, or the argmin of the
  // outstanding requests / allocated blocks as of each worker's last processed boundary; ties go
  // to the lowest worker index
  auto pick = [&](bool toD) -> u32 {
    const u32 cnt = toD ? Y : X;
    if (c.dispatch == OR_DISPATCH_RR) return (u32)((toD ? rrD++ : rrP++) % cnt);
    u32 best = 0;
    u64 bestv = UINT64_MAX;
    for (u32 w = 0; w < cnt; ++w) {
      u64 v;
      if (c.dispatch == OR_DISPATCH_LEAST_OUTSTANDING) {
        v = toD ? Dw[w].pending.size() + Dw[w].xfer.size() + Dw[w].R.size() + Dw[w].Q.size()
                : Pw[w].queue.size() + Pw[w].batch.size();
      } else {
        v = toD ? totD - Dw[w].free.size() : totP - Pw[w].free.size();
      }
      if (v < bestv) {
        bestv = v;
        best = w;
      }
    }
    return best;
  };

  while (true) {
    if (n_done == n) break;
    i64 td = arr < n ? req[arr].a : INF;  // next dispatch event
    for (const PW &w : Pw)
      if (!w.batch.empty()) td = std::min(td, w.tdisp);
    i64 tb = INF;  // next worker boundary
    for (const PW &w : Pw) tb = std::min(tb, w.t);
    for (const DW &w : Dw) tb = std::min(tb, w.t);
    const i64 tnext = std::min(td, tb);
    if (tnext == INF) {
      g_err = "P/D deadlock: every worker waits";
      delete run;
      return nullptr;
    }
    if (c.horizon_ns >= 0 && tnext >= c.horizon_ns) {
      S.status_flags |= 4;
      break;
    }
    if (td <= tb) {
      // ============================================================ dispatch events at td
      std::vector<u32> ids;
      std::vector<char> done_prefill;
      for (PW &w : Pw) {
        if (w.batch.empty() || w.tdisp != td) continue;
        ids.insert(ids.end(), w.batch.begin(), w.batch.end());
        w.batch.clear();
        w.tdisp = INF;
      }
      std::sort(ids.begin(), ids.end());
      const size_t n_comp = ids.size();
      while (arr < n && req[arr].a == td) ids.push_back(arr++);  // arrivals: larger ids
      for (size_t q = 0; q < ids.size(); ++q) {
        const u32 id = ids[q];
        NReq &x = req[id];
        if (q < n_comp) {  // end-of-prefill breakpoint: to a decode worker (o = 1 finished on P)
          if (x.status == 1) continue;
          const u32 j = pick(true);
          x.dw = j;
          x.join = td;
          Dw[j].pending.push_back(id);
          if (Dw[j].idle && td < Dw[j].t) Dw[j].t = td;
        } else {  // arrival: to a prefill worker
          const u32 i = pick(false);
          x.pw = i;
          Pw[i].queue.push_back(id);
          if (Pw[i].idle && td < Pw[i].t) Pw[i].t = td;
        }
      }
      continue;
    }
    // the worker to advance: earliest boundary, decode workers first, lower index first
    int wsel = -1;
    for (u32 j = 0; j < Y && wsel < 0; ++j)
      if (Dw[j].t == tb) wsel = (int)(X + j);
    for (u32 i = 0; i < X && wsel < 0; ++i)
      if (Pw[i].t == tb) wsel = (int)i;
    if (wsel >= (int)X) {
      // ================================================================ D_j boundary
      const u32 j = (u32)wsel - X;
      DW &w = Dw[j];
      const u32 wid = (u32)wsel;
      const i64 t = w.t;
      std::vector<u32> xv(w.xfer.begin(), w.xfer.end());
      for (u32 id : xv) {
        if (req[id].xend <= t) {
          w.xfer.erase(id);
          w.R.insert(id);
        }
      }
      std::map<u32, Kind> kind;
      const u64 F = w.free.size();
      std::vector<u32> Rv(w.R.begin(), w.R.end());
      auto need_of = [&](u32 id) -> u64 { return (req[id].ctx % bs == 0) ? 1 : 0; };
      u64 sum_need = 0;
      for (u32 id : Rv) sum_need += need_of(id);
      u64 m = 0, swap_out = 0;
      if (sum_need > F) {
        const u64 nr = Rv.size();
        for (m = 1; m <= nr; ++m) {
          u64 lhs = 0, rhs = F;
          for (u64 q = 0; q < nr - m; ++q) lhs += need_of(Rv[q]);
          for (u64 q = nr - m; q < nr; ++q) rhs += req[Rv[q]].dblocks.size();
          if (lhs <= rhs) break;
        }
        if (m > nr) {
          g_err = "P/D: no victim count satisfies c.4 step 3";
          delete run;
          return nullptr;
        }
        for (u64 q = 0; q < m; ++q) {
          const u32 id = Rv[nr - 1 - q];
          NReq &x = req[id];
          const u64 held = x.dblocks.size();
          for (u32 b : x.dblocks) {
            w.free.insert(b);
            ev(w.k, 2, wid, id, b);
          }
          x.dblocks.clear();
          x.n_preempt += 1;
          if (SWAPM) swap_out += held * dD.block_bytes;
          else x.ctx = 0;
          w.R.erase(id);
          w.Q.insert(id);
        }
        npre += m;
      }
      for (u32 id : w.R) {
        kind[id] = K_DEC;
        if (need_of(id)) {
          const u32 b = *w.free.begin();
          w.free.erase(w.free.begin());
          req[id].dblocks.push_back(b);
          ev(w.k, 1, wid, id, b);
        }
      }
      u64 n_res = 0, n_adm = 0, swap_in = 0, tokens = w.R.size();
      if (m == 0) {
        std::vector<u32> Qv(w.Q.begin(), w.Q.end());
        for (u32 id : Qv) {
          NReq &x = req[id];
          u64 need, tok;
          if (SWAPM) {
            need = ceil_div(x.ctx, bs) + ((x.ctx % bs == 0) ? 1 : 0);
            tok = 1;
          } else {
            need = ceil_div(x.p + x.gen, bs);
            tok = x.p + x.gen;
          }
          const bool ok = (w.R.size() + w.xfer.size() + 1 <= c.max_num_seqs) &&
                          (tokens + tok <= c.max_batched_tokens) &&
                          ((i64)w.free.size() - (i64)need >= (i64)c.watermark_blocks);
          if (!ok) break;
          for (u64 q = 0; q < need; ++q) {
            const u32 b = *w.free.begin();
            w.free.erase(w.free.begin());
            x.dblocks.push_back(b);
            ev(w.k, 1, wid, id, b);
          }
          w.Q.erase(id);
          w.R.insert(id);
          ++n_res;
          tokens += tok;
          if (SWAPM) {
            swap_in += ceil_div(x.ctx, bs) * dD.block_bytes;
            kind[id] = K_DEC;
          } else {
            kind[id] = K_PRE_RECOMP;
          }
        }
        // pull pending requests FCFS onto this worker's ingress link (reading R-X3)
        if (w.Q.empty() && (c.kind != OR_STATIC || (w.R.empty() && w.xfer.empty()))) {
          while (!w.pending.empty() && req[w.pending.front()].join <= t) {
            const u32 id = w.pending.front();
            NReq &x = req[id];
            const u64 need = ceil_div(x.p, bs);
            if (w.R.size() + w.xfer.size() + 1 > c.max_num_seqs) break;
            if ((i64)w.free.size() - (i64)need < (i64)c.watermark_blocks) break;
            for (u64 q = 0; q < need; ++q) {
              const u32 b = *w.free.begin();
              w.free.erase(w.free.begin());
              x.dblocks.push_back(b);
              ev(w.k, 1, wid, id, b);
            }
            const u64 bytes = (u64)x.p * dD.kvb;
            const double sec = (double)bytes * inv_link;
            const i64 dur = (i64)std::floor(sec * 1e9 + 0.5);
            const i64 start = std::max(t, w.link_busy);
            x.xend = start + dur;
            x.xstarted = true;
            w.link_busy = x.xend;
            w.xfer.insert(id);
            w.pending.pop_front();
            ++n_adm;
            ++n_xfer;
            xfer_bytes += bytes;
            PW &pw = Pw[x.pw];
            if (pw.idle && x.xend < pw.t) pw.t = x.xend;  // its prefill worker waits for these blocks
          }
        }
      }
      if (w.R.empty()) {  // nothing runnable: wait for a transfer end (dispatches wake it too)
        i64 wake = INF;
        for (u32 id : w.xfer) wake = std::min(wake, req[id].xend);
        for (u32 id : w.pending)
          if (req[id].join > t) wake = std::min(wake, req[id].join);
        w.t = wake;
        w.idle = true;
        continue;
      }
      std::vector<Prefill> pf;
      std::vector<u64> dec;
      u64 Np = 0, Cd = 0;
      for (u32 id : w.R) {
        const NReq &x = req[id];
        if (kind[id] == K_DEC) {
          dec.push_back(x.ctx + 1);
          Cd += x.ctx + 1;
        } else {
          pf.push_back({x.p + x.gen, 0});
          Np += x.p + x.gen;
        }
      }
      const i64 T = iter_time(KD.k, pf, dec, swap_out, swap_in);
      const i64 te = t + T;
      const u64 blocks = totD - w.free.size();
      const u64 entries = w.R.size();
      u64 n_fin = 0;
      std::vector<u32> Rc(w.R.begin(), w.R.end());
      for (u32 id : Rc) {
        NReq &x = req[id];
        if (kind[id] == K_PRE_RECOMP) {
          x.ctx = x.p + x.gen;
          x.gen += 1;
        } else {
          x.ctx += 1;
          x.gen += 1;
        }
        const i64 gap = te - x.last_tok;
        x.max_gap = std::max(x.max_gap, gap);
        x.last_tok = te;
        if (x.gen == x.o) {
          finish_req(id, te, w.k);
          for (u32 b : x.dblocks) {
            w.free.insert(b);
            ev(w.k, 2, wid, id, b);
          }
          x.dblocks.clear();
          w.R.erase(id);
          ++n_fin;
        }
      }
      sched_d += fold_sched(w.k | ((u64)wid << 40), (u64)t, (u64)T, pf.size(), dec.size(), Np, Cd, m, n_res, n_adm, 0,
                       n_fin, blocks);
      run->iters.push_back({w.k, t, T, pf.size(), dec.size(), Np, Cd, m, n_res, n_adm, 0, n_fin, blocks, wid, 0});
      req_iters += entries;
      w.peak = std::max(w.peak, blocks);
      w.bns += blocks * (u64)T;
      swo += swap_out;
      swi += swap_in;
      w.t = te;
      w.last = te;
      ++w.k;
      w.idle = false;
    } else {
      // ================================================================ P_i boundary
      const u32 i = (u32)wsel;
      PW &w = Pw[i];
      const i64 t = w.t;
      std::vector<u32> hv(w.holders.begin(), w.holders.end());
      for (u32 id : hv) {  // blocks of finished transfers come back (ascending id)
        NReq &x = req[id];
        if (!(x.xstarted && x.xend <= t)) continue;
        for (u32 b : x.pblocks) {
          w.free.insert(b);
          ev(w.k, 2, i, id, b);
        }
        x.pblocks.clear();
        w.holders.erase(id);
      }
      u64 tokens = 0, n_rej = 0;
      while (!w.queue.empty()) {
        const u32 id = w.queue.front();
        NReq &x = req[id];
        const u64 need = ceil_div(x.p, bs);
        if (need > totP - c.watermark_blocks) {
          x.status = 2;
          ++n_rej;
          ++n_done;
          w.queue.pop_front();
          continue;
        }
        if (w.batch.size() + 1 > c.max_num_seqs) break;
        if (tokens + x.p > c.max_batched_tokens) break;
        if ((i64)w.free.size() - (i64)need < (i64)c.watermark_blocks) break;
        for (u64 q = 0; q < need; ++q) {
          const u32 b = *w.free.begin();
          w.free.erase(w.free.begin());
          x.pblocks.push_back(b);
          ev(w.k, 1, i, id, b);
        }
        w.batch.push_back(id);
        tokens += x.p;
        w.queue.pop_front();
      }
      nrej_tot += n_rej;
      if (w.batch.empty()) {  // idle: wait for a dispatch or for P blocks to come back
        i64 wake = INF;
        for (u32 id : w.holders)
          if (req[id].xstarted) wake = std::min(wake, req[id].xend);
        w.t = wake;
        w.idle = true;
        continue;
      }
      std::vector<Prefill> pf;
      u64 Np = 0;
      for (u32 id : w.batch) {
        pf.push_back({req[id].p, 0});
        Np += req[id].p;
      }
      const i64 T = iter_time(KP.k, pf, {}, 0);
      const i64 te = t + T;
      const u64 blocks = totP - w.free.size();
      u64 n_fin = 0;
      for (u32 id : w.batch) {  // the first token at the end-of-prefill breakpoint
        NReq &x = req[id];
        x.ctx = x.p;
        x.gen = 1;
        x.first_tok = te;
        x.last_tok = te;
        if (x.gen == x.o) {
          finish_req(id, te, w.k);
          for (u32 b : x.pblocks) {
            w.free.insert(b);
            ev(w.k, 2, i, id, b);
          }
          x.pblocks.clear();
          ++n_fin;
        } else {
          w.holders.insert(id);
        }
      }
      sched_d += fold_sched(w.k | ((u64)i << 40), (u64)t, (u64)T, w.batch.size(), 0, Np, 0, 0, 0, w.batch.size(), n_rej,
                       n_fin, blocks);
      run->iters.push_back({w.k, t, T, w.batch.size(), 0, Np, 0, 0, 0, w.batch.size(), n_rej, n_fin, blocks, i, 0});
      req_iters += w.batch.size();
      w.tdisp = te;  // the batch goes to the global scheduler at te
      w.t = te;
      w.last = te;
      ++w.k;
      w.idle = false;
    }
    if (c.check_invariants) {
      bool ok = true;
      for (u32 q = 0; q < X; ++q) {
        u64 h = 0;
        for (u32 id = 0; id < n; ++id)
          if (req[id].pw == q) h += req[id].pblocks.size();
        ok &= h + Pw[q].free.size() == totP;
      }
      for (u32 q = 0; q < Y; ++q) {
        const DW &w = Dw[q];
        u64 h = 0;
        for (u32 id = 0; id < n; ++id)
          if (req[id].dw == q) h += req[id].dblocks.size();
        ok &= h + w.free.size() == totD;
        for (u32 id : w.R) ok &= req[id].dblocks.size() == ceil_div(req[id].ctx, bs) && req[id].dw == q;
        for (u32 id : w.xfer) ok &= req[id].dblocks.size() == ceil_div(req[id].p, bs) && req[id].dw == q;
        for (u32 id : w.Q) ok &= req[id].dblocks.empty();
      }
      if (!ok) {
        g_err = "P/D node invariant violated";
        delete run;
        return nullptr;
      }
    }
  }

  run->records.resize(n);
  u64 n_fin = 0;
  for (u32 i = 0; i < n; ++i) {
    const NReq &x = req[i];
    oracle_record &rec = run->records[i];
    rec.ttft_ns = (x.gen >= 1 || x.status == 1) ? x.first_tok - x.a : 0;
    rec.e2e_ns = x.status == 1 ? x.finish - x.a : 0;
    rec.mtpot_ns = x.status == 1 ? x.max_gap : 0;
    rec.n_preempt = x.n_preempt;
    rec.status = x.status;
    rec.finish_k = x.status == 1 ? x.finish_k : 0;
    if (x.status == 1) ++n_fin;
  }
  i64 t_final = 0;
  u64 kall = 0, peak = 0, bns = 0;
  for (const PW &w : Pw) {
    t_final = std::max(t_final, w.last);
    kall += w.k;
  }
  for (const DW &w : Dw) {
    t_final = std::max(t_final, w.last);
    kall += w.k;
    peak = std::max(peak, w.peak);
    bns += w.bns;
  }
  S.n_requests = n;
  S.n_finished = n_fin;
  S.n_rejected = nrej_tot;
  S.n_unfinished = n - n_fin - nrej_tot;
  if (nrej_tot == n) S.status_flags |= 2;
  S.n_iterations = kall;
  S.n_request_iterations = req_iters;
  S.n_preemptions = npre;
  S.swap_out_bytes = swo;
  S.swap_in_bytes = swi;
  S.t_final = t_final;
  S.sched_digest = sched_d;
  S.block_digest = block_d;
  S.request_digest = req_d;
  // the decode pool (reading R-X5): y workers' blocks; peak = the largest single-worker peak
  S.total_blocks = (u64)Y * totD;
  S.peak_blocks = peak;
  S.block_ns_sum = bns;
  S.mean_util = (t_final > 0 && totD > 0) ? (double)bns / ((double)S.total_blocks * (double)t_final) : 0.0;
  S.n_transfers = n_xfer;
  S.transfer_bytes = xfer_bytes;
  std::vector<Req> rr(n);
  for (u32 i = 0; i < n; ++i) {
    rr[i].a = req[i].a;
    rr[i].p = req[i].p;
    rr[i].o = req[i].o;
    rr[i].status = req[i].status;
    rr[i].first_tok = req[i].first_tok;
    rr[i].finish = req[i].finish;
    rr[i].max_gap = req[i].max_gap;
  }
  metrics(c, dD, rr, S);
  bool ovf = false;
  for (u32 w = 0; w < X + Y; ++w) build_trace(c, run->iters, w, t_final, run->trace[w], ovf);
  if (ovf) S.status_flags |= 1;
  return run;
}

// ----------------------------------------------------------------- NEXT-2 multi-round workload
// SURVEY §8(f) NEXT-2 and reading R-N2 in DESIGN.md.  num_requests conversations
// arrive as the a.1 Poisson stream (round 0 uses the a.1 draws).  Y2 gives the round count: top
// bit 0 -> 1 round (probability 1/2), else 2 + floor(low31 * 6 / 2^31) in {2..7}.  Round r >= 1
// draws Z = philox((c, 2, r, 0)): think gap -det_log(u(Z0, Z1)) * think_mean, new-turn prompt
// length from (Z2, Z3); W = philox((c, 3, r, 0)): output length from (W0, W1).  Its prompt is the
// prior context plus the new turn, P_r = P_{r-1} + o_{r-1} + q_r; a round with P_r + 1 > mml ends
// the conversation; o_r = min(o_r, mml - P_r).  Request rid = base_c + r, in conversation order.
struct Rounds {
  std::vector<i64> at;  // round 0: arrival; round r >= 1: think gap after round r-1 finishes
  std::vector<u32> P, O, conv;
  std::vector<u32> base, nr;
};

u32 draw_len(const oracle_cfg &c, bool prompt, u32 w0, u32 w1) {
  if (c.len_dist == OR_LEN_FIXED) return prompt ? c.prompt_a : c.output_a;
  if (c.len_dist == OR_LEN_UNIFORM) {
    const u32 a = prompt ? c.prompt_a : c.output_a, b = prompt ? c.prompt_b : c.output_b;
    return a + (u32)(((u64)w0 * (u64)(b - a + 1)) >> 32);
  }
  return prompt ? table_draw(c.pt_n, c.pt_lo, c.pt_hi, c.pt_thr, w0, w1)
                : table_draw(c.ot_n, c.ot_lo, c.ot_hi, c.ot_thr, w0, w1);
}

bool workload_rounds(const oracle_cfg &c, Rounds &W) {
  if (c.len_dist == OR_LEN_TRACE) return fail("multi-round workloads need generated lengths (not TRACE)");
  std::vector<i64> A;
  std::vector<u32> Pl, Ol;
  if (!workload(c, A, Pl, Ol)) return false;  // round 0 = the a.1 stream
  const u32 n = c.num_requests;
  const u32 key[2] = {(u32)(c.seed & 0xffffffffu), (u32)(c.seed >> 32)};
  const double think_ns = c.think_mean_s * 1e9;
  W = Rounds();
  W.base.assign(n, 0);
  W.nr.assign(n, 0);
  for (u32 i = 0; i < n; ++i) {
    const u32 cy[4] = {i, 1, 0, 0};
    u32 Y[4];
    philox(cy, key, Y);
    const u32 R = (Y[2] >> 31) == 0 ? 1u : 2u + (u32)(((u64)(Y[2] & 0x7fffffffu) * 6u) >> 31);
    W.base[i] = (u32)W.P.size();
    W.at.push_back(A[i]);
    W.P.push_back(Pl[i]);
    W.O.push_back(Ol[i]);
    W.conv.push_back(i);
    u64 prevP = Pl[i], prevO = Ol[i];
    u32 made = 1;
    for (u32 r = 1; r < R; ++r) {
      const u32 cz[4] = {i, 2, r, 0}, cw[4] = {i, 3, r, 0};
      u32 Z[4], Wd[4];
      philox(cz, key, Z);
      philox(cw, key, Wd);
      const u64 v = ((u64)Z[0] << 21) | (u64)(Z[1] >> 11);
      const double u = (double)(v + 1) * 0x1p-53;
      const double E = -det_log(u);
      const i64 gap = (i64)std::floor(E * think_ns + 0.5);
      const u64 q = draw_len(c, true, Z[2], Z[3]);
      u64 o = draw_len(c, false, Wd[0], Wd[1]);
      const u64 Pr = prevP + prevO + q;
      if (Pr + 1 > c.max_model_len) break;  // the context no longer fits: the conversation ends
      if (o > c.max_model_len - Pr) o = c.max_model_len - Pr;
      W.at.push_back(gap);
      W.P.push_back((u32)Pr);
      W.O.push_back((u32)o);
      W.conv.push_back(i);
      prevP = Pr;
      prevO = o;
      ++made;
    }
    W.nr[i] = made;
  }
  return true;
}

// ----------------------------------------------------------------- NEXT-2 simulation
// The c.4 unified loop (MIXED) over a dynamic request stream: round 0 of conversation c arrives
// at its a.1 time, round r >= 1 at (finish of round r-1) + its think gap.  Arrived requests queue
// FCFS by (arrival time, conversation); "id order" (victims, resumes, requesters) is arrival
// order.  With the memory cache: a finishing round stores its context (P + o - 1
// tokens with KV) for its conversation as the most recently used entry of a host LRU cache of
// capacity blocks (evicting least recently used entries); admitting round r >= 1 whose
// conversation is cached is a hit: its prefill is the (P - c0, c0) row with c0 = the cached
// tokens, the entry becomes most recently used, and the iteration pays 800 ns per cached block
// before the prefill.  Reading R-N2.
oracle_run *simulate_mr(const oracle_cfg &c) {
  if (c.iter_mode != OR_MIXED) {
    g_err = "multi-round workloads run MIXED iterations";
    return nullptr;
  }
  oracle_derived d;
  if (!derive(c, 0, d)) return nullptr;
  CostCtx K = cost_ctx(c, d, 0);
  Rounds Wr;
  if (!workload_rounds(c, Wr)) return nullptr;
  const u32 nconv = c.num_requests;
  const u32 n = (u32)Wr.P.size();
  const u64 bs = c.block_size, total = d.total_blocks;
  const bool SWAPM = c.preempt == OR_SWAP;
  const bool RATIO = c.kind == OR_CONT_RATIO;
  const bool CACHE = c.memory_cache != 0;
  const u64 cache_cap = c.cache_capacity_blocks ? c.cache_capacity_blocks : 4 * total;
  const double fetch_s = c.cache_fetch_ns_per_block * 1e-9;

  std::vector<Req> req(n);
  for (u32 i = 0; i < n; ++i) {
    req[i].p = Wr.P[i];
    req[i].o = Wr.O[i];
  }
  for (u32 cv = 0; cv < nconv; ++cv) req[Wr.base[cv]].a = Wr.at[Wr.base[cv]];  // round 0 arrivals are known
  oracle_run *run = new oracle_run();
  std::memset(&run->summary, 0, sizeof(run->summary));
  oracle_summary &S = run->summary;
  std::set<u32> freeset;
  for (u64 b = 0; b < total; ++b) freeset.insert((u32)b);
  std::vector<u32> seq2rid;        // arrival sequence -> request
  std::set<u32> R, Q;              // arrival sequence numbers
  std::deque<u32> waitq;           // arrived, not admitted (arrival sequence order)
  std::set<std::pair<i64, u32>> pend;  // follow-up rounds: (arrival time, conversation)
  std::vector<u32> next_round(nconv, 0);
  std::vector<u32> seq_of(n, 0);
  // host LRU cache: conversation -> cached tokens; front = least recently used
  std::list<u32> lru;
  std::map<u32, std::pair<u64, std::list<u32>::iterator>> cache;
  u64 cache_used = 0;
  u32 next0 = 0;  // next conversation whose round 0 has not arrived
  i64 t = 0;
  u64 k = 0;
  u32 n_done = 0;
  u64 sched_d = 0, block_d = 0, req_d = 0;
  u64 req_iters = 0, n_preempt_total = 0, swap_out_total = 0, swap_in_total = 0;
  u64 peak = 0, block_ns_sum = 0, n_rej_total = 0;

  auto alloc_lowest = [&](u32 rid, u64 cnt) {
    for (u64 j = 0; j < cnt; ++j) {
      const u32 b = *freeset.begin();
      freeset.erase(freeset.begin());
      req[rid].blocks.push_back(b);
      block_d += fold_block(k, 1, rid, b);
      if (c.keep_events) run->events.push_back({k, 1, rid, b, 0});
    }
  };
  auto free_all = [&](u32 rid) {
    for (u32 b : req[rid].blocks) {
      freeset.insert(b);
      block_d += fold_block(k, 2, rid, b);
      if (c.keep_events) run->events.push_back({k, 2, rid, b, 0});
    }
    req[rid].blocks.clear();
  };
  auto cache_touch = [&](u32 cv) {  // make most recently used
    auto it = cache.find(cv);
    lru.erase(it->second.second);
    lru.push_back(cv);
    it->second.second = std::prev(lru.end());
  };
  auto cache_store = [&](u32 cv, u64 tokens) {
    const u64 blk = ceil_div(tokens, bs);
    auto it = cache.find(cv);
    if (it != cache.end()) {
      cache_used -= ceil_div(it->second.first, bs);
      lru.erase(it->second.second);
      cache.erase(it);
    }
    if (blk > cache_cap) return;  // larger than the whole cache: not stored
    lru.push_back(cv);
    cache[cv] = {tokens, std::prev(lru.end())};
    cache_used += blk;
    while (cache_used > cache_cap) {  // evict least recently used
      const u32 ev = lru.front();
      lru.pop_front();
      cache_used -= ceil_div(cache[ev].first, bs);
      cache.erase(ev);
    }
  };
  // the next arrival: (time, conversation, round)
  auto next_arrival = [&](i64 &ta, u32 &cv) -> bool {
    ta = INT64_MAX;
    bool any = false;
    if (next0 < nconv) {
      ta = Wr.at[Wr.base[next0]];
      cv = next0;
      any = true;
    }
    if (!pend.empty()) {
      const auto &e = *pend.begin();
      if (!any || e.first < ta || (e.first == ta && e.second < cv)) {
        ta = e.first;
        cv = e.second;
        any = true;
      }
    }
    return any;
  };

  while (true) {
    if (n_done == n) break;
    if (c.horizon_ns >= 0 && t >= c.horizon_ns) {
      S.status_flags |= 4;
      break;
    }
    // 1. ingest: arrivals at or before t join the FCFS queue in (time, conversation) order
    {
      i64 ta;
      u32 cv;
      while (next_arrival(ta, cv) && ta <= t) {
        const u32 r = next_round[cv];
        const u32 rid = Wr.base[cv] + r;
        if (r == 0) ++next0;
        else pend.erase(pend.begin());
        req[rid].a = ta;
        seq_of[rid] = (u32)seq2rid.size();
        seq2rid.push_back(rid);
        waitq.push_back(seq_of[rid]);
      }
    }
    // 2. idle skip
    if (R.empty() && Q.empty() && waitq.empty()) {
      i64 ta;
      u32 cv;
      if (!next_arrival(ta, cv)) {
        g_err = "multi-round: nothing left to arrive but requests unresolved";
        delete run;
        return nullptr;
      }
      t = ta;
      continue;
    }
    std::map<u32, Kind> kind;  // by arrival sequence
    std::map<u32, u64> c0_of;  // cache-hit prefix of fresh entries
    u64 n_res = 0, n_adm = 0, n_rej = 0, swap_in = 0, m = 0, swap_out = 0, fetch_blocks = 0;
    // 3. decode reservation + preemption (victims: latest arrivals)
    const u64 F = freeset.size();
    std::vector<u32> Rv(R.begin(), R.end());
    auto rid_of = [&](u32 s) { return seq2rid[s]; };
    auto need_of = [&](u32 s) -> u64 { return (req[rid_of(s)].ctx % bs == 0) ? 1 : 0; };
    u64 sum_need = 0;
    for (u32 s : Rv) sum_need += need_of(s);
    if (sum_need > F) {
      const u64 nr = Rv.size();
      for (m = 1; m <= nr; ++m) {
        u64 lhs = 0, rhs = F;
        for (u64 j = 0; j < nr - m; ++j) lhs += need_of(Rv[j]);
        for (u64 j = nr - m; j < nr; ++j) rhs += req[rid_of(Rv[j])].blocks.size();
        if (lhs <= rhs) break;
      }
      if (m >= nr) {
        g_err = "preemption would evict r_1 (validation should make this impossible)";
        delete run;
        return nullptr;
      }
      for (u64 i = 0; i < m; ++i) {
        const u32 s = Rv[nr - 1 - i];
        Req &x = req[rid_of(s)];
        const u64 held = x.blocks.size();
        free_all(rid_of(s));
        x.n_preempt += 1;
        if (SWAPM) swap_out += held * d.block_bytes;
        else x.ctx = 0;
        R.erase(s);
        Q.insert(s);
      }
      n_preempt_total += m;
    }
    for (u32 s : R) {
      kind[s] = K_DEC;
      if (need_of(s)) alloc_lowest(rid_of(s), 1);
    }
    u64 tokens = R.size();
    if (m == 0) {
      // 4. resume, head first
      std::vector<u32> Qv(Q.begin(), Q.end());
      for (u32 s : Qv) {
        Req &x = req[rid_of(s)];
        u64 need, tok;
        if (SWAPM) {
          need = ceil_div(x.ctx, bs) + ((x.ctx % bs == 0) ? 1 : 0);
          tok = 1;
        } else {
          need = ceil_div(x.p + x.gen, bs);
          tok = x.p + x.gen;
        }
        const bool ok = (R.size() + 1 <= c.max_num_seqs) && (tokens + tok <= c.max_batched_tokens) &&
                        ((i64)freeset.size() - (i64)need >= (i64)c.watermark_blocks);
        if (!ok) break;
        alloc_lowest(rid_of(s), need);
        Q.erase(s);
        R.insert(s);
        ++n_res;
        tokens += tok;
        if (SWAPM) {
          swap_in += ceil_div(x.ctx, bs) * d.block_bytes;
          kind[s] = K_DEC;
        } else {
          kind[s] = K_PRE_RECOMP;
        }
      }
      // 5. fresh FCFS admission over the arrival queue, with cache lookups
      if (Q.empty() && (c.kind != OR_STATIC || R.empty())) {
        while (!waitq.empty()) {
          const u32 s = waitq.front();
          const u32 rid = rid_of(s);
          Req &x = req[rid];
          const u64 need = ceil_div(x.p, bs);
          const u64 cap = RATIO ? d.ratio_limit : total - c.watermark_blocks;
          if (need > cap) {  // rejected; its conversation's later rounds never arrive
            const u32 cv = Wr.conv[rid];
            const u32 last = Wr.base[cv] + Wr.nr[cv];
            for (u32 q = rid; q < last; ++q) {
              req[q].status = 2;
              ++n_rej;
              ++n_done;
            }
            waitq.pop_front();
            continue;
          }
          const u64 fr = freeset.size();
          if (R.size() + 1 > c.max_num_seqs) break;
          if (tokens + x.p > c.max_batched_tokens) break;
          if ((i64)fr - (i64)need < (i64)c.watermark_blocks) break;
          if (RATIO && (total - fr) + need > d.ratio_limit) break;
          alloc_lowest(rid, need);
          R.insert(s);
          kind[s] = K_PRE_FRESH;
          tokens += x.p;
          ++n_adm;
          waitq.pop_front();
          u64 c0 = 0;
          const u32 cv = Wr.conv[rid];
          if (CACHE && rid > Wr.base[cv]) {
            auto it = cache.find(cv);
            if (it != cache.end()) {  // hit
              c0 = it->second.first;
              fetch_blocks += ceil_div(c0, bs);
              cache_touch(cv);
            }
          }
          c0_of[s] = c0;
        }
      }
    }
    n_rej_total += n_rej;
    if (kind.empty()) continue;
    // 7. cost
    std::vector<Prefill> pf;
    std::vector<u64> dec;
    u64 Np = 0, Cd = 0;
    for (const auto &kv : kind) {
      const Req &x = req[rid_of(kv.first)];
      if (kv.second == K_DEC) {
        dec.push_back(x.ctx + 1);
        Cd += x.ctx + 1;
      } else if (kv.second == K_PRE_FRESH) {
        const u64 c0 = c0_of[kv.first];
        pf.push_back({x.p - c0, c0});
        Np += x.p - c0;
      } else {
        pf.push_back({x.p + x.gen, 0});
        Np += x.p + x.gen;
      }
    }
    const i64 T = iter_time(K, pf, dec, swap_out, swap_in, fetch_blocks, fetch_s);
    // 8. commit
    const i64 ts = t, te = t + T;
    const u64 blocks = total - freeset.size();
    const u64 entries = kind.size();
    u64 n_fin = 0;
    for (const auto &kv : kind) {
      const u32 s = kv.first;
      const u32 rid = rid_of(s);
      Req &x = req[rid];
      if (kv.second == K_PRE_FRESH) {
        x.ctx = x.p;
        x.gen = 1;
        x.first_tok = te;
        x.last_tok = te;
      } else {
        if (kv.second == K_PRE_RECOMP) {
          x.ctx = x.p + x.gen;
          x.gen += 1;
        } else {
          x.ctx += 1;
          x.gen += 1;
        }
        const i64 gap = te - x.last_tok;
        x.max_gap = std::max(x.max_gap, gap);
        x.last_tok = te;
      }
      if (x.gen == x.o) {
        x.status = 1;
        x.finish = te;
        x.finish_k = k;
        req_d += fold({rid, (u64)(x.first_tok - x.a), (u64)(x.finish - x.a), (u64)x.max_gap, x.n_preempt, k});
        free_all(rid);
        R.erase(s);
        ++n_fin;
        ++n_done;
        const u32 cv = Wr.conv[rid];
        if (CACHE) cache_store(cv, (u64)x.p + x.o - 1);
        const u32 r = rid - Wr.base[cv];
        if (r + 1 < Wr.nr[cv]) {
          next_round[cv] = r + 1;
          pend.insert({te + Wr.at[rid + 1], cv});
        }
      }
    }
    sched_d += fold_sched(k, (u64)ts, (u64)T, pf.size(), dec.size(), Np, Cd, m, n_res, n_adm, n_rej, n_fin, blocks);
    run->iters.push_back({k, ts, T, pf.size(), dec.size(), Np, Cd, m, n_res, n_adm, n_rej, n_fin, blocks, 0, 0});
    req_iters += entries;
    peak = std::max(peak, blocks);
    block_ns_sum += blocks * (u64)T;
    swap_out_total += swap_out;
    swap_in_total += swap_in;
    t = te;
    ++k;
    if (c.check_invariants) {
      std::set<u32> Rr, Qr;
      for (u32 s : R) Rr.insert(rid_of(s));
      for (u32 s : Q) Qr.insert(rid_of(s));
      if (!check_invariants(req, Rr, Qr, freeset, total, bs)) {
        delete run;
        return nullptr;
      }
      u64 used = 0;
      for (const auto &e : cache) used += ceil_div(e.second.first, bs);
      if (used != cache_used || cache_used > cache_cap) {
        g_err = "memory cache accounting";
        delete run;
        return nullptr;
      }
    }
  }

  run->records.resize(n);
  u64 n_fin = 0;
  for (u32 i = 0; i < n; ++i) {
    const Req &x = req[i];
    oracle_record &rec = run->records[i];
    rec.ttft_ns = (x.gen >= 1 || x.status == 1) ? x.first_tok - x.a : 0;
    rec.e2e_ns = x.status == 1 ? x.finish - x.a : 0;
    rec.mtpot_ns = x.status == 1 ? x.max_gap : 0;
    rec.n_preempt = x.n_preempt;
    rec.status = x.status;
    rec.finish_k = x.status == 1 ? x.finish_k : 0;
    if (x.status == 1) ++n_fin;
  }
  S.n_requests = n;
  S.n_finished = n_fin;
  S.n_rejected = n_rej_total;
  S.n_unfinished = n - n_fin - n_rej_total;
  if (n_rej_total == n) S.status_flags |= 2;
  S.n_iterations = k;
  S.n_request_iterations = req_iters;
  S.n_preemptions = n_preempt_total;
  S.swap_out_bytes = swap_out_total;
  S.swap_in_bytes = swap_in_total;
  S.t_final = t;
  S.sched_digest = sched_d;
  S.block_digest = block_d;
  S.request_digest = req_d;
  S.total_blocks = total;
  S.peak_blocks = peak;
  S.block_ns_sum = block_ns_sum;
  S.mean_util = (t > 0 && total > 0) ? (double)block_ns_sum / ((double)total * (double)t) : 0.0;
  metrics(c, d, req, S);
  bool ovf = false;
  build_trace(c, run->iters, 0, t, run->trace[0], ovf);
  if (ovf) S.status_flags |= 1;
  return run;
}

}  // namespace

// ======================================================================== C ABI
extern "C" {

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  philox(ctr, key, out);
}

double oracle_det_log(double u) { return det_log(u); }

int oracle_derive(const oracle_cfg *cfg, int decode_worker, oracle_derived *out) {
  return derive(*cfg, decode_worker, *out) ? 0 : -1;
}

int oracle_workload(const oracle_cfg *cfg, int64_t *arrival, uint32_t *prompt, uint32_t *output) {
  std::vector<i64> a;
  std::vector<u32> p, o;
  if (!workload(*cfg, a, p, o)) return -1;
  for (u32 i = 0; i < cfg->num_requests; ++i) {
    arrival[i] = a[i];
    prompt[i] = p[i];
    output[i] = o[i];
  }
  return 0;
}

int64_t oracle_iter_time_ns(const oracle_cfg *cfg, int decode_worker, uint32_t n_prefill,
                            const uint32_t *P, const uint32_t *c0, const uint32_t *emits,
                            uint32_t n_decode, const uint32_t *c, uint64_t swap_out, uint64_t swap_in) {
  oracle_derived d;
  if (!derive(*cfg, decode_worker, d)) return -1;
  const CostCtx K = cost_ctx(*cfg, d, decode_worker);
  std::vector<Prefill> pf;
  std::vector<u64> dec;
  for (u32 i = 0; i < n_prefill; ++i) pf.push_back({P[i], c0[i], emits ? emits[i] != 0 : true});
  for (u32 i = 0; i < n_decode; ++i) dec.push_back(c[i]);
  return iter_time(K, pf, dec, swap_out, swap_in);
}

int64_t oracle_workload_rounds(const oracle_cfg *cfg, int64_t *arrival_or_think, uint32_t *prompt,
                               uint32_t *output, uint32_t *conv) {
  g_err.clear();
  Rounds W;
  if (!workload_rounds(*cfg, W)) return -1;
  for (size_t i = 0; i < W.P.size(); ++i) {
    if (arrival_or_think) arrival_or_think[i] = W.at[i];
    if (prompt) prompt[i] = W.P[i];
    if (output) output[i] = W.O[i];
    if (conv) conv[i] = W.conv[i];
  }
  return (int64_t)W.P.size();
}

double oracle_pipeline(uint64_t n_chunks, double a, double b, uint64_t slots) {
  return pipeline(n_chunks, a, b, slots);
}

uint64_t oracle_fold(const uint64_t *fields, uint32_t n) {
  u64 h = 0x9E3779B97F4A7C15ull;
  for (u32 i = 0; i < n; ++i) h = mix(h ^ fields[i]);
  return h;
}

oracle_run *oracle_simulate(const oracle_cfg *cfg) {
  g_err.clear();
  if (cfg->multi_round) {
    if (cfg->topology != OR_UNIFIED) {
      g_err = "multi-round workloads run on the unified topology";
      return nullptr;
    }
    return simulate_mr(*cfg);
  }
  if (cfg->topology == OR_PD_PAIR) {
    const bool one = (cfg->n_prefill <= 1 && cfg->n_decode <= 1);
    return (one && !cfg->force_general) ? simulate_pd(*cfg) : simulate_pdn(*cfg);
  }
  return simulate_unified(*cfg);
}

const char *oracle_error(void) { return g_err.c_str(); }

void oracle_summary_get(const oracle_run *r, oracle_summary *out) { *out = r->summary; }

uint64_t oracle_records(const oracle_run *r, oracle_record *out) {
  if (out) std::copy(r->records.begin(), r->records.end(), out);
  return r->records.size();
}
uint64_t oracle_iters(const oracle_run *r, oracle_iter *out) {
  if (out) std::copy(r->iters.begin(), r->iters.end(), out);
  return r->iters.size();
}
uint64_t oracle_trace(const oracle_run *r, int worker, oracle_sample *out) {
  static const std::vector<oracle_sample> empty;
  const std::vector<oracle_sample> &v = (worker >= 0 && worker < OR_MAX_WORKERS) ? r->trace[worker] : empty;
  if (out) std::copy(v.begin(), v.end(), out);
  return v.size();
}
uint64_t oracle_events(const oracle_run *r, oracle_event *out) {
  if (out) std::copy(r->events.begin(), r->events.end(), out);
  return r->events.size();
}
void oracle_free(oracle_run *r) { delete r; }

}  // extern "C"
