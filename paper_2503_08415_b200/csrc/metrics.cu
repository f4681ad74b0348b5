// metrics.cu -- a.8 metrics: exact nearest-rank quantiles by MSD radix
// select, means, throughput/goodput and the 384-B summary record.
// PAPER.md: P50/P99/max latency P:321; CDFs P:323; normalized latency P:429; TTFT and
// mTPOT SLO goodput P:458-465.
#include "dev_common.cuh"

namespace ts {

// ------------------------------------------------------------------ a.8 metrics
// Metric value (seconds, fp64) of request i if it belongs to the metric's sample set.
__device__ __forceinline__ bool metric_value(u32 metric, const tokensim_request_record &r, u32 o, double &v) {
  if (r.status != TOKENSIM_REQ_FINISHED) return false;
  switch (metric) {
    case TOKENSIM_TTFT: v = __ddiv_rn(__ll2double_rn(r.ttft_ns), 1e9); return true;
    case TOKENSIM_E2E: v = __ddiv_rn(__ll2double_rn(r.e2e_ns), 1e9); return true;
    case TOKENSIM_MTPOT: v = __ddiv_rn(__ll2double_rn(r.mtpot_ns), 1e9); return true;
    case TOKENSIM_TPOT:
      if (o < 2) return false;
      v = __ddiv_rn(__ddiv_rn(__ll2double_rn(r.e2e_ns - r.ttft_ns), __uint2double_rn(o - 1)), 1e9);
      return true;
    default:  // NORM
      v = __ddiv_rn(__ddiv_rn(__ll2double_rn(r.e2e_ns), __uint2double_rn(o)), 1e9);
      return true;
  }
}

struct SelShared {
  u32 hist[256];
  u32 cnt;
  u32 digit, rem;
  u64 red[32];
  u32 hist3[3][256];  // block_select3: one histogram per distinct target prefix
  u32 digit3[3], rem3[3];
};

// Exact rank-th smallest (1-based) of keys[0..cnt) by MSD radix select, 8 bits per pass,
// starting below the bytes shared by min and max.  Block-wide; returns on all threads.
__device__ u64 block_select(const u64 *keys, u32 cnt, u32 rank, u64 kmin, u64 kmax, SelShared &sh) {
  const u32 tid = threadIdx.x, nt = blockDim.x;
  const u64 diff = kmin ^ kmax;
  if (diff == 0) return kmin;
  int top = 63 - __clzll((long long)diff);
  int shift = (top / 8) * 8;
  u64 mask = shift + 8 >= 64 ? 0ull : ~((1ull << (shift + 8)) - 1ull);
  u64 prefix = kmin & mask;
  u32 rem = rank;
  for (; shift >= 0; shift -= 8) {
    for (u32 x = tid; x < 256; x += nt) sh.hist[x] = 0;
    __syncthreads();
    for (u32 x = tid; x < cnt; x += nt) {
      const u64 kk = keys[x];
      if ((kk & mask) == prefix) atomicAdd(&sh.hist[(kk >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns bins [8l, 8l+8)
      u32 loc[8], s = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        loc[q] = sh.hist[tid * 8 + q];
        s += loc[q];
      }
      const u32 incl = scan_incl(s);
      const u32 excl = incl - s;
      const u32 hit = __ballot_sync(FULLMASK, incl >= rem);
      const u32 L = (u32)(__ffs(hit) - 1);
      if (tid == L) {
        u32 c = excl;
        u32 d = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (c + loc[q] >= rem) {
            d = tid * 8 + q;
            break;
          }
          c += loc[q];
        }
        sh.digit = d;
        sh.rem = rem - c;
      }
    }
    __syncthreads();
    prefix |= (u64)sh.digit << shift;
    mask |= 255ull << shift;
    rem = sh.rem;
    __syncthreads();
  }
  return prefix;
}

// The rank[0..3)-th smallest keys in one set of MSD passes (ranks ascending, so the targets'
// prefixes are ordered; targets with the same prefix share a histogram).  Same digits as three
// block_select calls, a third of the passes over the keys.
__device__ void block_select3(const u64 *keys, u32 cnt, const u32 rank[3], u64 kmin, u64 kmax, SelShared &sh,
                              u64 out[3]) {
  const u32 tid = threadIdx.x, nt = blockDim.x;
  const u64 diff = kmin ^ kmax;
  if (diff == 0) {
    out[0] = out[1] = out[2] = kmin;
    return;
  }
  int top = 63 - __clzll((long long)diff);
  int shift = (top / 8) * 8;
  u64 mask = shift + 8 >= 64 ? 0ull : ~((1ull << (shift + 8)) - 1ull);
  u64 pre[3];
  u32 rem[3];
  for (int t = 0; t < 3; ++t) {
    pre[t] = kmin & mask;
    rem[t] = rank[t];
  }
  for (; shift >= 0; shift -= 8) {
    // histogram index of each target: the first target with the same prefix
    const u32 h1 = pre[1] == pre[0] ? 0u : 1u;
    const u32 h2 = pre[2] == pre[1] ? h1 : 2u;
    for (u32 x = tid; x < 3 * 256; x += nt) (&sh.hist3[0][0])[x] = 0;
    __syncthreads();
    for (u32 x = tid; x < cnt; x += nt) {
      const u64 kk = keys[x];
      const u64 km = kk & mask;
      const u32 bin = (u32)(kk >> shift) & 255u;
      if (km == pre[0]) atomicAdd(&sh.hist3[0][bin], 1u);
      else if (km == pre[1]) atomicAdd(&sh.hist3[h1][bin], 1u);
      else if (km == pre[2]) atomicAdd(&sh.hist3[h2][bin], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      for (int t = 0; t < 3; ++t) {
        const u32 h = t == 0 ? 0u : t == 1 ? h1 : h2;
        u32 loc[8], sm = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          loc[q] = sh.hist3[h][tid * 8 + q];
          sm += loc[q];
        }
        const u32 incl = scan_incl(sm);
        const u32 excl = incl - sm;
        const u32 hit = __ballot_sync(FULLMASK, incl >= rem[t]);
        const u32 L = (u32)(__ffs(hit) - 1);
        if (tid == L) {
          u32 c = excl, d = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (c + loc[q] >= rem[t]) {
              d = tid * 8 + q;
              break;
            }
            c += loc[q];
          }
          sh.digit3[t] = d;
          sh.rem3[t] = rem[t] - c;
        }
      }
    }
    __syncthreads();
    for (int t = 0; t < 3; ++t) {
      pre[t] |= (u64)sh.digit3[t] << shift;
      rem[t] = sh.rem3[t];
    }
    mask |= 255ull << shift;
    __syncthreads();
  }
  for (int t = 0; t < 3; ++t) out[t] = pre[t];
}

__device__ u64 block_reduce_u64(u64 v, bool is_max, SelShared &sh) {
  const u32 tid = threadIdx.x, w = tid >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (u32 o = 16; o; o >>= 1) {
    const u64 y = __shfl_xor_sync(FULLMASK, v, o);
    v = is_max ? (y > v ? y : v) : v + y;
  }
  __syncthreads();
  if ((tid & 31) == 0) sh.red[w] = v;
  __syncthreads();
  u64 r = is_max ? 0ull : 0ull;
  for (u32 q = 0; q < nw; ++q) r = is_max ? (sh.red[q] > r ? sh.red[q] : r) : r + sh.red[q];
  __syncthreads();
  return r;
}
__device__ u64 block_reduce_min(u64 v, SelShared &sh) {
  const u32 tid = threadIdx.x, w = tid >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (u32 o = 16; o; o >>= 1) {
    const u64 y = __shfl_xor_sync(FULLMASK, v, o);
    v = y < v ? y : v;
  }
  __syncthreads();
  if ((tid & 31) == 0) sh.red[w] = v;
  __syncthreads();
  u64 r = ~0ull;
  for (u32 q = 0; q < nw; ++q) r = sh.red[q] < r ? sh.red[q] : r;
  __syncthreads();
  return r;
}

// Build the key array of one metric (order irrelevant); returns count.
__device__ u32 build_keys(u32 metric, const tokensim_request_record *rec, const u32 *OU, u32 n, u64 *keys,
                          SelShared &sh, u64 &kmin, u64 &kmax) {
  if (threadIdx.x == 0) sh.cnt = 0;
  __syncthreads();
  u64 mn = ~0ull, mx = 0;
  for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
    const tokensim_request_record r = rec[i];
    double v;
    if (metric_value(metric, r, OU[i], v)) {
      const u64 key = (u64)__double_as_longlong(v);  // v >= 0: bit patterns order like values
      const u32 slot = atomicAdd(&sh.cnt, 1u);
      keys[slot] = key;
      mn = key < mn ? key : mn;
      mx = key > mx ? key : mx;
    }
  }
  __syncthreads();
  const u32 cnt = sh.cnt;
  kmin = block_reduce_min(mn, sh);
  kmax = block_reduce_u64(mx, true, sh);
  return cnt;
}

__device__ __forceinline__ u32 nearest_rank(u32 q_bp, u32 cnt) {
  u64 r = ((u64)q_bp * cnt + 9999) / 10000;
  return r < 1 ? 1u : (u32)r;
}

__global__ void __launch_bounds__(256) summary_kernel(SweepParams P, u64 *scratch, u32 smem_keys) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ SelShared sh;
  const u64 j = blockIdx.x;
  const u64 point = P.begin + j * P.stride;
  const Coords cd = decode_point(point, P.n_pol, P.n_rates, P.n_seeds);
  const u32 g = P.group_of_point_mode ? 0u : cd.rate * P.n_seeds + cd.seed;
  const u32 n = P.n_req;
  const i64 *A = P.arrival + (size_t)g * n;
  const u32 *OU = P.output + (size_t)g * n;
  const tokensim_request_record *rec = P.rec + (size_t)j * n;
  u64 *keys = n <= smem_keys ? reinterpret_cast<u64 *>(dsm) : scratch + (size_t)j * n;
  const SimStats st = P.stats[j];
  const i64 slo_t = P.slo_ttft_ns, slo_m = P.slo_mtpot_ns;

  // counts for goodput, sums for integer means
  u64 g_mt = 0, g_both = 0, s_ttft = 0, s_e2e = 0, s_mt = 0, dig_r = 0;
  for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
    const tokensim_request_record r = rec[i];
    if (r.status != TOKENSIM_REQ_FINISHED) continue;
    // request digest (c.6): fold(id, ttft, e2e, mtpot, n_preempt, finish_k), wrapping sum
    u64 h = FOLD_INIT;
    h = mix64(h ^ (u64)i);
    h = mix64(h ^ (u64)r.ttft_ns);
    h = mix64(h ^ (u64)r.e2e_ns);
    h = mix64(h ^ (u64)r.mtpot_ns);
    h = mix64(h ^ (u64)r.n_preempt);
    h = mix64(h ^ (u64)r.finish_iter);
    dig_r += h;
    s_ttft += (u64)r.ttft_ns;
    s_e2e += (u64)r.e2e_ns;
    s_mt += (u64)r.mtpot_ns;
    if (r.mtpot_ns <= slo_m) {
      ++g_mt;
      if (r.ttft_ns <= slo_t) ++g_both;
    }
  }
  g_mt = block_reduce_u64(g_mt, false, sh);
  g_both = block_reduce_u64(g_both, false, sh);
  s_ttft = block_reduce_u64(s_ttft, false, sh);
  s_e2e = block_reduce_u64(s_e2e, false, sh);
  s_mt = block_reduce_u64(s_mt, false, sh);
  dig_r = block_reduce_u64(dig_r, false, sh);
  // sequential fp64 sums for TPOT / NORM in ascending id (SURVEY c.6): the terms (two fp64
  // divisions each) are formed by all threads into the key buffer, then one thread adds them in
  // id order; excluded requests contribute +0.0, which leaves a running sum >= +0 unchanged
  __shared__ double seq_tp, seq_norm;
  double *term = reinterpret_cast<double *>(keys);
  for (u32 pass = 0; pass < 2; ++pass) {
    for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
      const tokensim_request_record r = rec[i];
      const u32 o = OU[i];
      double v = 0.0;
      if (r.status == TOKENSIM_REQ_FINISHED) {
        if (pass == 0) {
          if (o >= 2) v = __ddiv_rn(__ll2double_rn(r.e2e_ns - r.ttft_ns), __uint2double_rn(o - 1));
        } else {
          v = __ddiv_rn(__ll2double_rn(r.e2e_ns), __uint2double_rn(o));
        }
      }
      term[i] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0;
#pragma unroll 8
      for (u32 i = 0; i < n; ++i) a = __dadd_rn(a, term[i]);
      if (pass == 0) seq_tp = a;
      else seq_norm = a;
    }
    __syncthreads();
  }
  tokensim_summary S;
  const u64 nfin = st.n_finished;
  const u32 qbp[4] = {5000, 9000, 9900, 10000};
  for (u32 m = 0; m < 5; ++m) {
    u64 kmin, kmax;
    const u32 cnt = build_keys(m, rec, OU, n, keys, sh, kmin, kmax);
    u64 sel[3] = {0, 0, 0};
    if (cnt) {
      const u32 rk[3] = {nearest_rank(qbp[0], cnt), nearest_rank(qbp[1], cnt), nearest_rank(qbp[2], cnt)};
      block_select3(keys, cnt, rk, kmin, kmax, sh, sel);
    }
    for (u32 qi = 0; qi < 4; ++qi)
      S.stat[m][qi] = cnt ? __longlong_as_double((long long)(qi == 3 ? kmax : sel[qi])) : 0.0;
    double mean = 0.0;
    if (cnt) {
      const double dn = __ull2double_rn(cnt);
      if (m == TOKENSIM_TTFT) mean = __ddiv_rn(__ddiv_rn(__ll2double_rn((i64)s_ttft), dn), 1e9);
      if (m == TOKENSIM_E2E) mean = __ddiv_rn(__ddiv_rn(__ll2double_rn((i64)s_e2e), dn), 1e9);
      if (m == TOKENSIM_MTPOT) mean = __ddiv_rn(__ddiv_rn(__ll2double_rn((i64)s_mt), dn), 1e9);
      if (m == TOKENSIM_TPOT) mean = __ddiv_rn(__ddiv_rn(seq_tp, dn), 1e9);
      if (m == TOKENSIM_NORM) mean = __ddiv_rn(__ddiv_rn(seq_norm, dn), 1e9);
    }
    S.stat[m][4] = mean;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    S.version = 1;
    S.status_flags = st.flags;
    S.point = point;
    const u64 nreq = P.multi_round ? st.n_req : (u64)n;  // multi-round: this point's rounds
    S.n_requests = nreq;
    S.n_finished = nfin;
    S.n_rejected = st.n_rejected;
    S.n_unfinished = nreq - nfin - st.n_rejected;
    S.n_iterations = st.n_iterations;
    S.n_request_iterations = st.n_req_iters;
    S.n_preemptions = st.n_preempt;
    S.swap_out_bytes = st.swap_out;
    S.swap_in_bytes = st.swap_in;
    S.first_arrival_ns = n ? A[0] : 0;
    S.last_finish_ns = st.last_finish;
    S.sched_digest = st.sched_d;
    S.block_digest = st.block_d;
    S.request_digest = dig_r;
    S.total_blocks = (u32)st.total_blocks;
    S.peak_blocks = (u32)st.peak_blocks;
    S.mean_util = (st.t_final > 0 && st.total_blocks > 0)
                      ? __ddiv_rn(__ull2double_rn(st.block_ns_sum),
                                  __dmul_rn(__ull2double_rn(st.total_blocks), __ll2double_rn(st.t_final)))
                      : 0.0;
    const i64 span = st.last_finish - S.first_arrival_ns;
    S.throughput_rps = S.goodput_mtpot_rps = S.goodput_both_rps = 0.0;
    if (nfin > 0 && span > 0) {
      const double sec = __ddiv_rn(__ll2double_rn(span), 1e9);
      S.throughput_rps = __ddiv_rn(__ull2double_rn(nfin), sec);
      S.goodput_mtpot_rps = __ddiv_rn(__ull2double_rn(g_mt), sec);
      S.goodput_both_rps = __ddiv_rn(__ull2double_rn(g_both), sec);
    }
    S.t_final_ns = st.t_final;
    S.block_ns_sum = st.block_ns_sum;
    P.summ[j] = S;
  }
}

cudaError_t launch_summary(const SweepParams &p, cudaStream_t st) {
  if (p.n_run == 0) return cudaSuccess;
  const u32 smem_keys = kSummarySmemKeys;  // 96 KB of keys in shared memory; else workspace scratch
  const size_t smem = p.n_req <= smem_keys ? (size_t)p.n_req * 8 : 0;
  cudaError_t e = cudaFuncSetAttribute(summary_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem_keys * 8));
  if (e != cudaSuccess) return e;
  summary_kernel<<<(unsigned)p.n_run, 256, smem, st>>>(p, p.scratch, smem_keys);
  return cudaGetLastError();
}

// Arbitrary nearest-rank quantiles of one (point, metric): d_ranks holds q_bp values.
__global__ void __launch_bounds__(256) quantile_kernel(SweepParams P, u64 j, u32 metric, const u32 *q_bp,
                                                       u32 n_q, double *out, u64 *keys) {
  __shared__ SelShared sh;
  const u64 point = P.begin + j * P.stride;
  const Coords cd = decode_point(point, P.n_pol, P.n_rates, P.n_seeds);
  const u32 g = P.group_of_point_mode ? 0u : cd.rate * P.n_seeds + cd.seed;
  const u32 n = P.n_req;
  const u32 *OU = P.output + (size_t)g * n;
  const tokensim_request_record *rec = P.rec + (size_t)j * n;
  u64 kmin, kmax;
  const u32 cnt = build_keys(metric, rec, OU, n, keys, sh, kmin, kmax);
  for (u32 q = 0; q < n_q; ++q) {
    double v = 0.0;
    if (cnt) v = __longlong_as_double((long long)block_select(keys, cnt, nearest_rank(q_bp[q], cnt), kmin, kmax, sh));
    if (threadIdx.x == 0) out[q] = v;
    __syncthreads();
  }
}

cudaError_t launch_quantiles(const SweepParams &p, u64 j, u32 metric, const u32 *d_ranks, u32 n_q,
                             double *d_out, u64 *d_keys, cudaStream_t st) {
  quantile_kernel<<<1, 256, 0, st>>>(p, j, metric, d_ranks, n_q, d_out, d_keys);
  return cudaGetLastError();
}

}  // namespace ts
