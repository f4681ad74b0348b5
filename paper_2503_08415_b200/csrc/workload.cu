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
  // multi-round (NEXT-2): this is round 0 of every conversation, expanded by rounds_kernel
  const u32 n = P.multi_round ? P.n_conv : P.n_req;
  i64 *A = (P.multi_round ? P.mr_a0 : P.arrival) + (size_t)g * n;
  u32 *PRm = (P.multi_round ? P.mr_p0 : P.prompt) + (size_t)g * n;
  u32 *OUt = (P.multi_round ? P.mr_o0 : P.output) + (size_t)g * n;
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

// ------------------------------------------------------------------ NEXT-2 rounds
// SURVEY §8(f) NEXT-2, reading R-N2: Y2 of round 0 gives the round count (top bit
// 0: one round; else 2 + floor(low31 * 6 / 2^31)); round r >= 1 of conversation c draws
// Z = philox(c, 2, r, 0) -- think gap from (Z0, Z1), new turn from (Z2, Z3) -- and
// W = philox(c, 3, r, 0) -- output from (W0, W1).  P_r = P_{r-1} + o_{r-1} + turn; a round
// with P_r + 1 > mml ends the conversation; o_r = min(o_r, mml - P_r).
__device__ __forceinline__ u32 draw_len_dev(const SweepParams &P, bool prompt, u32 w0, u32 w1) {
  if (P.len_dist == TOKENSIM_LEN_FIXED) return prompt ? P.prompt_a : P.output_a;
  if (P.len_dist == TOKENSIM_LEN_UNIFORM) {
    const u32 a = prompt ? P.prompt_a : P.output_a, b = prompt ? P.prompt_b : P.output_b;
    return a + (u32)(((u64)w0 * (u64)(b - a + 1)) >> 32);
  }
  return table_draw(prompt ? P.pt : P.ot, w0, w1);
}
// round r >= 1 of conversation c after (prevP, prevO): false if it does not fit
__device__ __forceinline__ bool next_round_dev(const SweepParams &P, u32 c, u32 r, u32 k0, u32 k1, u32 prevP,
                                               u32 prevO, i64 &gap, u32 &Pr, u32 &Or) {
  u32 Z[4], Wd[4];
  philox4x32_10(c, 2, r, 0, k0, k1, Z);
  philox4x32_10(c, 3, r, 0, k0, k1, Wd);
  const u64 v = ((u64)Z[0] << 21) | (u64)(Z[1] >> 11);
  const double u = __dmul_rn(__ull2double_rn(v + 1), 0x1p-53);
  const double E = -det_log_dev(u);
  gap = (i64)floor(__dadd_rn(__dmul_rn(E, P.think_ns), 0.5));
  const u64 q = draw_len_dev(P, true, Z[2], Z[3]);
  u64 o = draw_len_dev(P, false, Wd[0], Wd[1]);
  const u64 p = (u64)prevP + prevO + q;
  if (p + 1 > P.M.mml) return false;
  if (o > P.M.mml - p) o = P.M.mml - p;
  Pr = (u32)p;
  Or = (u32)o;
  return true;
}
__device__ __forceinline__ u32 round_count_dev(u32 c, u32 k0, u32 k1) {
  u32 Y[4];
  philox4x32_10(c, 1, 0, 0, k0, k1, Y);
  return (Y[2] >> 31) == 0 ? 1u : 2u + (u32)(((u64)(Y[2] & 0x7fffffffu) * 6u) >> 31);
}
// One CTA per group: rounds per conversation, a block scan for the first rid of each, then the
// request-indexed arrays.
__global__ void __launch_bounds__(256) rounds_kernel(SweepParams P) {
  const u32 g = blockIdx.x;
  const u64 seed = P.seeds[g % P.n_seeds];
  const u32 k0 = (u32)(seed & 0xffffffffull), k1 = (u32)(seed >> 32);
  const u32 nc = P.n_conv, ns = P.n_req;
  const i64 *A0 = P.mr_a0 + (size_t)g * nc;
  const u32 *P0 = P.mr_p0 + (size_t)g * nc, *O0 = P.mr_o0 + (size_t)g * nc;
  u32 *BASE = P.mr_base + (size_t)g * nc, *NR = P.mr_nr + (size_t)g * nc;
  i64 *A = P.arrival + (size_t)g * ns;
  u32 *PR = P.prompt + (size_t)g * ns, *OU = P.output + (size_t)g * ns, *CV = P.mr_conv + (size_t)g * ns;
  __shared__ u32 wsum[8];
  __shared__ u32 carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const u32 lane = lane_id(), w = threadIdx.x >> 5;
  for (u32 base = 0; base < nc; base += 256) {
    const u32 c = base + threadIdx.x;
    u32 nr = 0;
    if (c < nc) {
      const u32 R = round_count_dev(c, k0, k1);
      u32 pp = P0[c], oo = O0[c];
      nr = 1;
      for (u32 r = 1; r < R; ++r) {
        i64 gap;
        u32 Pr, Or;
        if (!next_round_dev(P, c, r, k0, k1, pp, oo, gap, Pr, Or)) break;
        pp = Pr;
        oo = Or;
        ++nr;
      }
    }
    u32 x = scan_incl(nr);
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    u32 off = carry_s;
    for (u32 q = 0; q < w; ++q) off += wsum[q];
    if (c < nc) {
      const u32 b = off + x - nr;
      BASE[c] = b;
      NR[c] = nr;
      A[b] = A0[c];
      PR[b] = P0[c];
      OU[b] = O0[c];
      CV[b] = c;
      u32 pp = P0[c], oo = O0[c];
      for (u32 r = 1; r < nr; ++r) {
        i64 gap;
        u32 Pr, Or;
        next_round_dev(P, c, r, k0, k1, pp, oo, gap, Pr, Or);
        A[b + r] = gap;
        PR[b + r] = Pr;
        OU[b + r] = Or;
        CV[b + r] = c;
        pp = Pr;
        oo = Or;
      }
    }
    __syncthreads();
    if (threadIdx.x == 255) carry_s = off + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) P.mr_ntot[g] = carry_s;
}

cudaError_t launch_workload(const SweepParams &p, cudaStream_t st) {
  if (p.n_groups == 0) return cudaSuccess;
  workload_kernel<<<p.n_groups, 256, 0, st>>>(p);
  if (p.multi_round) rounds_kernel<<<p.n_groups, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace ts
