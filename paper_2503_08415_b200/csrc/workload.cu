// workload.cu -- a.1 workload generation: Philox4x32-10 counters per
// (seed, request), exponential gaps through det_log, integer table draws for lengths.
// PAPER.md: workloads "from datasets and parameters" P:214; QPS-driven request stream P:321.
#include "dev_common.cuh"

namespace ts {

// ------------------------------------------------------------------ a.1 generator
__device__ __forceinline__ void philox4x32_10(u32 c0, u32 c1, u32 c2, u32 c3, u32 k0, u32 k1,
                                              u32 out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const u32 lo0 = c0 * 0xD2511F53u, hi0 = __umulhi(c0, 0xD2511F53u);
    const u32 lo1 = c2 * 0xCD9E8D57u, hi1 = __umulhi(c2, 0xCD9E8D57u);
    const u32 n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// ln(u) for u in (0,1], normal: frexp by bit manipulation, ln(m) = 2 atanh(s) by a
// 13-term series in z = s^2 (SURVEY c.2); explicit RN intrinsics, fixed order.
__device__ __forceinline__ double det_log_dev(double u) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(u);
  int e = (int)((b >> 52) & 0x7ffull) - 1022;
  double m = __longlong_as_double((long long)((b & 0x800FFFFFFFFFFFFFull) | (0x3FEull << 52)));
  if (m < 0x1.6a09e667f3bcdp-1) {
    m = __dmul_rn(m, 2.0);
    e = e - 1;
  }
  const double s = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
  const double z = __dmul_rn(s, s);
  double p = __ddiv_rn(1.0, 25.0);
#pragma unroll
  for (int k = 11; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, z), __ddiv_rn(1.0, (double)(2 * k + 1)));
  const double LN2 = 0x1.62e42fefa39efp-1;
  return __dadd_rn(__dmul_rn((double)e, LN2), __dmul_rn(__dmul_rn(2.0, s), p));
}

__device__ __forceinline__ u32 table_draw(const u32 *t, u32 x, u32 y) {
  const u32 nb = t[0];
  const u32 *lo = t + 1, *hi = t + 1 + nb, *thr = t + 1 + 2 * nb;
  u32 b = nb - 1;
  for (u32 i = 0; i + 1 < nb; ++i) {
    if (x < thr[i]) {
      b = i;
      break;
    }
  }
  return lo[b] + (u32)(((u64)y * (u64)(hi[b] - lo[b])) >> 32);
}

// One CTA per (rate, seed) group; 256 threads; chunks of 256 requests with a carried
// block-wide inclusive prefix sum of the gaps (a_i = sum_{k<=i} gap_k).
__global__ void __launch_bounds__(256) workload_kernel(SweepParams P) {
  const u32 g = blockIdx.x;
  const u32 rate_i = g / P.n_seeds, seed_i = g % P.n_seeds;
  const double rate = P.rates[rate_i];
  const u64 seed = P.seeds[seed_i];
  const u32 k0 = (u32)(seed & 0xffffffffull), k1 = (u32)(seed >> 32);
  const double scale_ns = __ddiv_rn(1e9, rate);
  const u32 n = P.n_req;
  i64 *A = P.arrival + (size_t)g * n;
  u32 *PRm = P.prompt + (size_t)g * n;
  u32 *OUt = P.output + (size_t)g * n;
  __shared__ i64 wsum[8];
  __shared__ i64 carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const u32 lane = lane_id(), w = threadIdx.x >> 5;
  for (u32 base = 0; base < n; base += 256) {
    const u32 i = base + threadIdx.x;
    i64 gap = 0;
    if (i < n) {
      u32 X[4], Y[4];
      philox4x32_10(i, 0, 0, 0, k0, k1, X);
      philox4x32_10(i, 1, 0, 0, k0, k1, Y);
      const u64 v = ((u64)X[0] << 21) | (u64)(X[1] >> 11);
      const double u = __dmul_rn(__ull2double_rn(v + 1), 0x1p-53);
      const double E = -det_log_dev(u);
      gap = (i64)floor(__dadd_rn(__dmul_rn(E, scale_ns), 0.5));
      u32 pl = 0, ol = 0;
      if (P.len_dist == TOKENSIM_LEN_FIXED) {
        pl = P.prompt_a;
        ol = P.output_a;
      } else if (P.len_dist == TOKENSIM_LEN_UNIFORM) {
        pl = P.prompt_a + (u32)(((u64)X[2] * (u64)(P.prompt_b - P.prompt_a + 1)) >> 32);
        ol = P.output_a + (u32)(((u64)Y[0] * (u64)(P.output_b - P.output_a + 1)) >> 32);
      } else {  // TABLE (SHAREGPT_SYNTH_V1 is a TABLE the host filled in)
        pl = table_draw(P.pt, X[2], X[3]);
        ol = table_draw(P.ot, Y[0], Y[1]);
      }
      const u32 room = P.M.mml - pl;
      if (ol > room) ol = room;
      PRm[i] = pl;
      OUt[i] = ol;
    }
    // block inclusive scan of gap
    i64 x = gap;
#pragma unroll
    for (u32 o = 1; o < 32; o <<= 1) {
      const i64 y = __shfl_up_sync(FULLMASK, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    i64 off = carry_s;
    for (u32 q = 0; q < w; ++q) off += wsum[q];
    if (i < n) A[i] = off + x;
    __syncthreads();
    if (threadIdx.x == 255) carry_s = off + x;
    __syncthreads();
  }
}

cudaError_t launch_workload(const SweepParams &p, cudaStream_t st) {
  if (p.n_groups == 0) return cudaSuccess;
  workload_kernel<<<p.n_groups, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace ts
