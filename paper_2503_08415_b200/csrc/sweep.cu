// sweep.cu -- sm_100a kernels of the batched design-space sweep.
//
//   workload_kernel  (a.1)   one CTA per (rate, seed) group: Philox4x32-10 -> det_log ->
//                            exponential gaps -> block prefix sum -> arrivals; table lengths.
//   sim_kernel       (a.2-a.7) persistent; ONE WARP PER POINT pulled from an atomic
//                            longest-first queue.  Running/queued request slots, the free-block
//                            bitmap and the block-table slot pool live in shared memory; the
//                            per-slot work is lane-parallel (32 slots per warp step) with
//                            ballot/popc/prefix-scan for FCFS admission, the closed-form victim
//                            count, and lowest-free-first block extraction.
//   summary_kernel   (a.8)   one CTA per point: exact nearest-rank quantiles by MSD radix
//                            select, means, throughput/goodput, 384-B summary pack.
//
// Semantics: SURVEY.md §8(c) (c.1-c.6) under the readings in DESIGN.md -- the same text
// the CPU oracle (oracle/) follows; the two share no code.  Every fp64 operation uses
// explicit round-to-nearest intrinsics (__dadd_rn/__dmul_rn/__ddiv_rn) in the normative
// order, so no FMA contraction can occur (also compiled with --fmad=false).
//
// Paper anchors: worker loop with default end-of-iteration breakpoint P:243;
// continuous/static batching P:166-169; PagedAttention blocks P:172-173, P:274;
// preemption P:456-457; max-memory-ratio admission P:460; per-operator roofline
// compute simulator P:216; metrics P:321; memory over time
// P:552-565.
#include <cuda_runtime.h>

#include <cstdint>

#include "ts_internal.cuh"

namespace ts {

#define FULLMASK 0xffffffffu

// ------------------------------------------------------------------ warp primitives
__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ u32 scan_incl(u32 x) {
  const u32 l = lane_id();
#pragma unroll
  for (u32 o = 1; o < 32; o <<= 1) {
    u32 y = __shfl_up_sync(FULLMASK, x, o);
    if (l >= o) x += y;
  }
  return x;
}
__device__ __forceinline__ u64 warp_sum64(u64 x) {
#pragma unroll
  for (u32 o = 16; o; o >>= 1) x += __shfl_xor_sync(FULLMASK, x, o);
  return x;
}
__device__ __forceinline__ u64 shfl64(u64 x, u32 src) { return __shfl_sync(FULLMASK, x, src); }
__device__ __forceinline__ i64 shfl64i(i64 x, u32 src) { return __shfl_sync(FULLMASK, x, src); }

// r-th (0-based) set bit of w (r < popc(w))
__device__ __forceinline__ u32 select_bit(u32 w, u32 r) {
  u32 pos = 0;
#pragma unroll
  for (u32 s = 16; s; s >>= 1) {
    const u32 c = __popc(w & ((1u << s) - 1u));
    if (r >= c) {
      r -= c;
      pos += s;
      w >>= s;
    }
  }
  return pos;
}
// keep w without its `tk` lowest set bits (tk <= popc(w))
__device__ __forceinline__ u32 clear_lowest(u32 w, u32 tk, u32 c) {
  if (tk == 0) return w;
  if (tk >= c) return 0u;
  return w & ~((1u << select_bit(w, tk)) - 1u);
}

// ------------------------------------------------------------------ c.6 digests
__device__ __forceinline__ u64 mix64(u64 x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
#define FOLD_INIT 0x9E3779B97F4A7C15ull
__device__ __forceinline__ u64 fold4(u64 a, u64 b, u64 c, u64 d) {
  u64 h = FOLD_INIT;
  h = mix64(h ^ a);
  h = mix64(h ^ b);
  h = mix64(h ^ c);
  h = mix64(h ^ d);
  return h;
}

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

// ------------------------------------------------------------------ a.6 cost model
__device__ __forceinline__ double roof(u64 F, u64 B, double invF, double invB) {
  return fmax(__dmul_rn(__ull2double_rn(F), invF), __dmul_rn(__ull2double_rn(B), invB));
}

// T_ns for a batch given exact integer aggregates (SURVEY c.5; c0 = 0 so K_p = N_p).
__device__ __forceinline__ i64 iter_time_ns(const DevModel &M, const DevHw &H, u64 Np, u64 Ap, u64 Sp,
                                            u64 D, u64 Cd, u64 swap_bytes) {
  const u64 N = Np + D, S = Sp + D;
  double tQKV = 0.0, tATTP = 0.0, tATTD = 0.0, tO = 0.0, tUP = 0.0, tDOWN = 0.0, tLM = 0.0;
  if (N > 0) {
    tQKV = roof(2 * N * M.hq2g, M.s * (M.hq2g + N * M.h + N * M.q2g), H.invF, H.invB);
    tO = roof(2 * N * M.qh, M.s * (M.qh + N * M.q + N * M.h), H.invF, H.invB);
    tUP = roof(2 * N * M.hfu, M.s * (M.hfu + N * M.h + N * M.fu), H.invF, H.invB);
    tDOWN = roof(2 * N * M.fh, M.s * (M.fh + N * M.f + N * M.h), H.invF, H.invB);
  }
  if (Np > 0) tATTP = roof(4 * M.q * Ap, M.s * (Np * M.att_tok + M.g2 * Np), H.invF, H.invB);
  if (D > 0) tATTD = roof(4 * M.q * Cd, M.s * (D * M.att_tok + M.g2 * Cd), H.invF, H.invB);
  if (S > 0) tLM = roof(2 * S * M.Vh, M.s * (M.Vh + S * M.h + S * M.V), H.invF, H.invB);
  const double tl =
      __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(tQKV, tATTP), tATTD), tO), tUP), tDOWN);
  double T = __dmul_rn(tl, __ull2double_rn(M.L));
  T = __dadd_rn(T, tLM);
  if (H.tp > 1) {
    const u64 bar = 2 * (u64)(H.tp - 1) * N * M.h * M.s;
    T = __dadd_rn(T, __dmul_rn(__dmul_rn(__ull2double_rn(bar), H.invT), __ull2double_rn(2 * M.L)));
  }
  if (swap_bytes > 0) T = __dadd_rn(T, __dmul_rn(__ull2double_rn(swap_bytes), H.invH));
  T = __dadd_rn(T, H.overhead);
  return (i64)floor(__dadd_rn(__dmul_rn(T, 1e9), 0.5));
}

// ------------------------------------------------------------------ per-warp shared memory
struct WarpSmem {
  u32 *id, *ctx, *rem, *info;       // info: bt slot (bits 0-15) | n_preempt (bits 16-31)
  i64 *last, *maxgap, *arr, *ttft;  // last token time, max gap, arrival, ttft
  u32 *req_cum, *req_pt;            // block-requester list: cumulative count; pos | tpos<<10
  u32 *btfree;                      // cap/32 words, bit = free block-table slot
  u32 *bitmap;                      // free-block bitmap, bit = free block
};

__host__ __device__ inline size_t smem_per_warp_bytes(u32 cap, u32 nwords_max) {
  size_t b = (size_t)cap * (4 * 4 + 8 * 4 + 4 * 2) + (size_t)(cap / 32) * 4 + (size_t)nwords_max * 4;
  return (b + 15) & ~(size_t)15;
}
size_t sim_smem_per_warp(int cap, u32 nwords_max) { return smem_per_warp_bytes((u32)cap, nwords_max); }

__device__ __forceinline__ WarpSmem carve(unsigned char *base, u32 cap) {
  WarpSmem S;
  i64 *p64 = reinterpret_cast<i64 *>(base);
  S.last = p64;
  S.maxgap = p64 + cap;
  S.arr = p64 + 2 * cap;
  S.ttft = p64 + 3 * cap;
  u32 *p32 = reinterpret_cast<u32 *>(p64 + 4 * cap);
  S.id = p32;
  S.ctx = p32 + cap;
  S.rem = p32 + 2 * cap;
  S.info = p32 + 3 * cap;
  S.req_cum = p32 + 4 * cap;
  S.req_pt = p32 + 5 * cap;
  S.btfree = p32 + 6 * cap;
  S.bitmap = p32 + 6 * cap + cap / 32;
  return S;
}

// ------------------------------------------------------------------ a.5 allocator
// Return `held` blocks of table `tbl` (logical order is irrelevant to the bitmap; the
// block digest is an order-free sum) and lower the lowest-free-word hint.
__device__ __forceinline__ void free_blocks(u32 *bitmap, const u32 *tbl, u32 held, u32 id, u64 k,
                                            u64 &dig_b, u32 &hint) {
  u32 mn = 0xffffffffu;
  for (u32 x = lane_id(); x < held; x += 32) {
    const u32 b = tbl[x];
    atomicOr(&bitmap[b >> 5], 1u << (b & 31u));
    dig_b += fold4(k, 2, id, b);
    mn = min(mn, b >> 5);
  }
  mn = __reduce_min_sync(FULLMASK, mn);
  hint = min(hint, mn);
}

// Hand out the K lowest free blocks, in order, to the E requesters listed in S.req_*
// (entry e owns order indices [req_cum[e-1], req_cum[e]) and writes them to its block
// table from position tpos).  Equivalent to serving the requesters one after another
// with "take the lowest free block" (SURVEY c.4 step 3-5, reading A14).
__device__ bool alloc_ordered(const WarpSmem &S, u32 E, u32 K, u32 *bt, u32 btl, u64 k, u64 &dig_b,
                              u32 &hint, u32 nwords) {
  const u32 lane = lane_id();
  u32 o_base = 0, w = hint;
  while (o_base < K) {
    if (w >= nwords) return false;
    const u32 wi = w + lane;
    u32 word = wi < nwords ? S.bitmap[wi] : 0u;
    const u32 c = __popc(word);
    const u32 cum = scan_incl(c);
    const u32 tot = __shfl_sync(FULLMASK, cum, 31);
    if (tot == 0) {
      w += 32;
      continue;
    }
    const u32 take = min(tot, K - o_base);
    const u32 before = cum - c;
    for (u32 r0 = 0; r0 < take; r0 += 32) {
      const u32 idx = r0 + lane;
      const bool act = idx < take;
      const u32 tgt = act ? idx : 0u;
      u32 lo = 0;
#pragma unroll
      for (u32 s = 16; s; s >>= 1) {
        const u32 v = __shfl_sync(FULLMASK, cum, lo + s - 1);
        if (v <= tgt) lo += s;
      }
      const u32 wv = __shfl_sync(FULLMASK, word, lo);
      const u32 bv = __shfl_sync(FULLMASK, before, lo);
      if (act) {
        const u32 blk = (w + lo) * 32 + select_bit(wv, tgt - bv);
        const u32 o = o_base + idx;
        u32 a = 0, bnd = E;
        while (a < bnd) {
          const u32 mid = (a + bnd) >> 1;
          if (S.req_cum[mid] <= o) a = mid + 1;
          else bnd = mid;
        }
        const u32 start = a ? S.req_cum[a - 1] : 0u;
        const u32 pt = S.req_pt[a];
        const u32 pos = pt & 1023u;
        const u32 tpos = (pt >> 10) + (o - start);
        const u32 slot = S.info[pos] & 0xffffu;
        bt[(size_t)slot * btl + tpos] = blk;
        dig_b += fold4(k, 1, S.id[pos], blk);
      }
    }
    const u32 tk = take > before ? min(c, take - before) : 0u;
    if (tk && wi < nwords) {
      word = clear_lowest(word, tk, c);
      S.bitmap[wi] = word;
    }
    o_base += take;
    if (o_base < K) {
      w += 32;
    } else {
      const u32 nz = __ballot_sync(FULLMASK, word != 0u);
      w = nz ? w + (u32)(__ffs(nz) - 1) : w + 32;
    }
  }
  hint = w;
  __syncwarp();
  return true;
}

// Give `cnt` lanes (take=1, rank 0..cnt-1) the lowest free block-table slots.
__device__ __forceinline__ u32 alloc_btslots(u32 *btfree, u32 nw, bool take, u32 rank, u32 cnt) {
  const u32 lane = lane_id();
  u32 word = lane < nw ? btfree[lane] : 0u;
  const u32 c = __popc(word);
  const u32 cum = scan_incl(c);
  const u32 before = cum - c;
  const u32 tgt = take ? rank : 0u;
  u32 lo = 0;
#pragma unroll
  for (u32 s = 16; s; s >>= 1) {
    const u32 v = __shfl_sync(FULLMASK, cum, lo + s - 1);
    if (v <= tgt) lo += s;
  }
  const u32 wv = __shfl_sync(FULLMASK, word, lo);
  const u32 bv = __shfl_sync(FULLMASK, before, lo);
  const u32 slot = lo * 32 + select_bit(wv, tgt - bv);
  const u32 tk = cnt > before ? min(c, cnt - before) : 0u;
  if (tk && lane < nw) btfree[lane] = clear_lowest(word, tk, c);
  __syncwarp();
  return slot;
}

__device__ __forceinline__ void write_record(tokensim_request_record *r, i64 ttft, i64 e2e, i64 mt,
                                             u32 npre, u32 status, u32 fin_k) {
  ulonglong2 *q = reinterpret_cast<ulonglong2 *>(r);
  q[0] = make_ulonglong2((unsigned long long)ttft, (unsigned long long)e2e);
  const u64 w3 = (u64)(npre & 0xffffu) | ((u64)(status & 0xffu) << 16) | ((u64)fin_k << 32);
  q[1] = make_ulonglong2((unsigned long long)mt, (unsigned long long)w3);
}

// ------------------------------------------------------------------ a.2-a.7 one point
// Everything below is executed by all 32 lanes of the warp; scalar state is kept
// lane-uniform in registers; per-slot work is strided over lanes.
template <int CAP>
__device__ void simulate_unified(const SweepParams &P, u64 j, const WarpSmem &S, u32 *bt) {
  static_assert(CAP % 32 == 0 && CAP <= 1024, "CAP");
  const u32 lane = lane_id();
  const u32 ltm = lanemask_lt();
  const u64 point = P.begin + j * P.stride;
  const Coords cd = decode_point(point, P.n_pol, P.n_rates, P.n_seeds);
  const DevModel &M = P.M;
  const DevHw H = P.hw[cd.hw];
  const DevHP HP = P.hp[(size_t)cd.hw * P.n_pol + cd.pol];
  const DevPol PL = P.pol[cd.pol];
  const u32 g = P.group_of_point_mode ? 0u : cd.rate * P.n_seeds + cd.seed;
  const u32 n = P.n_req;
  const i64 *A = P.arrival + (size_t)g * n;
  const u32 *PR = P.prompt + (size_t)g * n;
  const u32 *OU = P.output + (size_t)g * n;
  tokensim_request_record *rec = P.rec + (size_t)j * n;
  tokensim_mem_sample *trc = P.trace + (size_t)j * 2 * P.trace_cap;
  tokensim_iter_record *itr = P.itrec + (size_t)j * P.it_cap;
  const u32 bs = PL.bs;
  const bool SWAPM = PL.preempt == TOKENSIM_SWAP;
  const bool RATIO = PL.kind == TOKENSIM_CONT_RATIO;
  const bool STATICP = PL.kind == TOKENSIM_STATIC;
  const u64 total = HP.total_blocks;
  const u32 nwords = HP.nwords;
  const u32 btl = P.bt_len;
  const u32 mns = PL.mns, mbt = PL.mbt;
  const i64 wm = (i64)PL.wm;

  // ---- init: records, bitmap, slot pool
  {
    ulonglong2 *r2 = reinterpret_cast<ulonglong2 *>(rec);
    const ulonglong2 z = make_ulonglong2(0ull, 0ull);
    for (u32 x = lane; x < 2 * n; x += 32) r2[x] = z;
    const u32 full_words = (u32)(total >> 5), tail = (u32)(total & 31u);
    for (u32 w = lane; w < nwords; w += 32)
      S.bitmap[w] = w < full_words ? 0xffffffffu : (w == full_words && tail ? ((1u << tail) - 1u) : 0u);
    for (u32 w = lane; w < CAP / 32; w += 32) S.btfree[w] = 0xffffffffu;
    __syncwarp();
  }

  i64 t = 0;
  u64 k = 0;
  u32 arr = 0, adm = 0, nR = 0, nQ = 0;
  u64 nfree = total;
  u32 hint = 0;
  u64 dig_s = 0, dig_b = 0, dig_r = 0;  // per-lane partial digests
  u64 req_iters = 0, npre = 0, swo_tot = 0, swi_tot = 0, nrej_tot = 0, nfin_tot = 0, peak = 0, bns = 0;
  i64 last_fin = 0;
  u32 flags = 0;
  // sched-field buffer: lane (k mod 32) holds iteration k's fields until the flush
  i64 b_t = 0, b_T = 0;
  u64 b_np = 0, b_cd = 0;
  u32 b_k = 0, b_blk = 0, b_spd = 0, b_mres = 0, b_adfin = 0, b_rej = 0;
  bool b_valid = false;
  auto flush_sched = [&]() {
    if (b_valid) {
      u64 h = FOLD_INIT;
      h = mix64(h ^ (u64)b_k);
      h = mix64(h ^ (u64)b_t);
      h = mix64(h ^ (u64)b_T);
      h = mix64(h ^ (u64)(b_spd & 0xffffu));
      h = mix64(h ^ (u64)(b_spd >> 16));
      h = mix64(h ^ b_np);
      h = mix64(h ^ b_cd);
      h = mix64(h ^ (u64)(b_mres & 0xffffu));
      h = mix64(h ^ (u64)(b_mres >> 16));
      h = mix64(h ^ (u64)(b_adfin & 0xffffu));
      h = mix64(h ^ (u64)b_rej);
      h = mix64(h ^ (u64)(b_adfin >> 16));
      h = mix64(h ^ (u64)b_blk);
      dig_s += h;
      if ((u64)b_k < P.it_cap) {
        tokensim_iter_record ir;
        ir.k = b_k;
        ir.t_start_ns = b_t;
        ir.T_ns = b_T;
        ir.n_prefill = b_spd & 0xffffu;
        ir.n_decode = b_spd >> 16;
        ir.N_p = b_np;
        ir.C_d = b_cd;
        ir.n_preempted = b_mres & 0xffffu;
        ir.n_resumed = b_mres >> 16;
        ir.n_admitted = b_adfin & 0xffffu;
        ir.n_rejected = b_rej;
        ir.n_finished = b_adfin >> 16;
        ir.blocks_in_use = b_blk;
        ir.worker = 0;
        ir.pad = 0;
        itr[b_k] = ir;
      }
    }
    b_valid = false;
  };
  // memory trace state (lane-uniform)
  const bool BINNED = P.trace_mode == TOKENSIM_TRACE_BINNED;
  const bool FULLT = P.trace_mode == TOKENSIM_TRACE_FULL;
  const i64 W = (i64)P.bin_ns;
  u64 tn = 0, bin = 0, acc_bns = 0;
  i64 bin_end = W;
  u32 acc_max = 0, acc_nit = 0;
  auto flush_bin = [&]() {
    if (tn < P.trace_cap) {
      if (lane == 0) {
        tokensim_mem_sample s;
        s.t_ns = (i64)bin * W;
        s.dur_ns = W;
        s.block_ns = acc_bns;
        s.blocks_max = acc_max;
        s.n_iter = acc_nit;
        trc[tn] = s;
      }
    } else {
      flags |= TOKENSIM_PT_TRACE_OVERFLOW;
    }
    ++tn;
    ++bin;
    bin_end += W;
    acc_bns = 0;
    acc_max = 0;
    acc_nit = 0;
  };

  // arrival window: lane l holds A[win + l]
  u32 win = 0;
  i64 wa = lane < n ? A[lane] : INT64_MAX;

  while (true) {
    // 0. termination
    if (adm == n && nR == 0 && nQ == 0) break;
    if (P.horizon >= 0 && t >= P.horizon) {
      flags |= TOKENSIM_PT_HORIZON_HIT;
      break;
    }
    // 1. ingest: a_i <= t become visible at this boundary
    while (arr < n) {
      if (arr >= win + 32) {
        win = arr;
        wa = win + lane < n ? A[win + lane] : INT64_MAX;
      }
      const u32 m = __ballot_sync(FULLMASK, (win + lane >= arr) && (wa <= t));
      arr += __popc(m);
      if (arr < win + 32) break;
    }
    // 2. idle skip
    if (nR == 0 && nQ == 0 && adm == arr) {
      t = shfl64i(wa, arr - win);
      continue;
    }
    // 3. decode reservation + preemption
    u32 sumneed = 0;
    for (u32 b0 = 0; b0 < nR; b0 += 32) {
      const u32 jj = b0 + lane;
      const bool need = jj < nR && (S.ctx[jj] % bs == 0);
      sumneed += __popc(__ballot_sync(FULLMASK, need));
    }
    u32 m = 0;
    u64 swap_out = 0;
    if ((u64)sumneed > nfree) {
      // minimal m with sum_{j<=n-m} need_j <= F + sum_{j>n-m} held_j (SURVEY c.4 step 3)
      u64 Sn = sumneed, Hh = 0;
      do {
        ++m;
        const u32 c = S.ctx[nR - m];
        Sn -= (c % bs == 0) ? 1 : 0;
        Hh += (c + bs - 1) / bs;
      } while (Sn > nfree + Hh);
      for (u32 v = nR - m; v < nR; ++v) {  // victims: latest arrivals (reading A7)
        const u32 c = S.ctx[v];
        const u32 held = (c + bs - 1) / bs;
        const u32 slot = S.info[v] & 0xffffu;
        free_blocks(S.bitmap, bt + (size_t)slot * btl, held, S.id[v], k, dig_b, hint);
        nfree += held;
        if (SWAPM) swap_out += (u64)held * HP.block_bytes;
        __syncwarp();
        if (lane == 0) {
          S.info[v] += 1u << 16;
          if (!SWAPM) S.ctx[v] = 0;
        }
      }
      __syncwarp();
      nR -= m;
      nQ += m;
      npre += m;
    }
    const u32 nR3 = nR;
    // surviving requests needing a block, ascending id -> requester list
    u32 E = 0, K = 0;
    for (u32 b0 = 0; b0 < nR; b0 += 32) {
      const u32 jj = b0 + lane;
      const u32 c = jj < nR ? S.ctx[jj] : 1u;
      const bool need = jj < nR && (c % bs == 0);
      const u32 bal = __ballot_sync(FULLMASK, need);
      if (need) {
        const u32 e = E + __popc(bal & ltm);
        S.req_cum[e] = e + 1;
        S.req_pt[e] = jj | ((c / bs) << 10);
      }
      E += __popc(bal);
    }
    K = E;
    nfree -= E;
    u32 nres = 0, nadm = 0, nrej = 0;
    u64 swap_in = 0, tokens = nR;
    if (m == 0) {
      // 4. resume, head first, stop at the first misfit
      if (nQ > 0) {
        u64 cum_need = 0, cum_tok = 0;
        for (u32 b0 = 0; b0 < nQ; b0 += 32) {
          const u32 jj = nR3 + b0 + lane;
          const bool valid = b0 + lane < nQ;
          u32 need = 0, tok = 0, held0 = 0;
          if (valid) {
            if (SWAPM) {
              const u32 c = S.ctx[jj];
              need = (c + bs - 1) / bs + ((c % bs == 0) ? 1u : 0u);
              tok = 1;
              held0 = (c + bs - 1) / bs;
            } else {
              const u32 id = S.id[jj];
              const u32 Pq = PR[id] + (OU[id] - S.rem[jj]);  // p + gen
              need = (Pq + bs - 1) / bs;
              tok = Pq;
            }
          }
          const u32 cn = scan_incl(need), ct = scan_incl(tok);
          const bool ok = valid && ((u64)nR3 + b0 + lane + 1 <= (u64)mns) &&
                          (tokens + cum_tok + ct <= (u64)mbt) &&
                          ((i64)nfree - (i64)(cum_need + cn) >= wm);
          const u32 okm = __ballot_sync(FULLMASK, ok);
          const u32 cnt = (~okm == 0u) ? 32u : (u32)(__ffs(~okm) - 1);
          if (lane < cnt) {
            S.req_cum[E + lane] = K + cn;
            S.req_pt[E + lane] = jj;
            if (!SWAPM) S.ctx[jj] = tok;  // recompute prefill of P = p + gen; ctx after commit
          }
          const u64 sw = warp_sum64(lane < cnt ? (u64)held0 : 0ull);
          if (cnt) {
            const u32 sn = __shfl_sync(FULLMASK, cn, cnt - 1), stk = __shfl_sync(FULLMASK, ct, cnt - 1);
            cum_need += sn;
            cum_tok += stk;
            K += sn;
            E += cnt;
            nres += cnt;
            if (SWAPM) swap_in += sw * HP.block_bytes;
          }
          if (cnt < 32) break;
        }
        nfree -= cum_need;
        tokens += cum_tok;
        nR += nres;
        nQ -= nres;
        __syncwarp();
      }
      // 5. fresh FCFS admission
      if (nQ == 0 && (!STATICP || nR == 0)) {
        while (adm < arr) {
          const u32 i = adm + lane;
          const bool valid = i < arr;
          const u32 p = valid ? PR[i] : 0u;
          const u32 o = valid ? OU[i] : 0u;
          const i64 a = valid ? A[i] : 0;
          const u32 need = (p + bs - 1) / bs;
          const bool rej = valid && (u64)need > HP.cap_fresh;
          const bool el = valid && !rej;
          const u32 ce = scan_incl(el ? 1u : 0u);
          const u32 cneed = scan_incl(el ? need : 0u);
          const u32 cp = scan_incl(el ? p : 0u);
          const bool ok = el && ((u64)nR + ce <= (u64)mns) && (tokens + cp <= (u64)mbt) &&
                          ((i64)nfree - (i64)cneed >= wm) &&
                          (!RATIO || (total - nfree) + cneed <= HP.ratio_limit);
          const u32 failm = __ballot_sync(FULLMASK, el && !ok);
          const u32 nvalid = min(32u, arr - adm);
          const u32 stop = failm ? (u32)(__ffs(failm) - 1) : nvalid;
          const bool take = el && lane < stop;
          const bool rj = rej && lane < stop;
          const u32 takem = __ballot_sync(FULLMASK, take);
          const u32 cnt = __popc(takem);
          if (cnt) {
            const u32 rank = __popc(takem & ltm);
            const u32 slot = alloc_btslots(S.btfree, CAP / 32, take, rank, cnt);
            if (take) {
              const u32 pos = nR + rank;
              S.id[pos] = i;
              S.ctx[pos] = p;  // fresh prefill of P = p; ctx after commit
              S.rem[pos] = o;
              S.info[pos] = slot;
              S.last[pos] = 0;
              S.maxgap[pos] = 0;
              S.arr[pos] = a;
              S.ttft[pos] = 0;
              S.req_cum[E + rank] = K + cneed;
              S.req_pt[E + rank] = pos;
            }
          }
          if (rj) reinterpret_cast<uint8_t *>(rec + i)[26] = (uint8_t)TOKENSIM_REQ_REJECTED;
          const u32 nrj = __popc(__ballot_sync(FULLMASK, rj));
          if (stop) {
            const u32 sneed = __shfl_sync(FULLMASK, cneed, stop - 1);
            const u32 sp = __shfl_sync(FULLMASK, cp, stop - 1);
            nfree -= sneed;
            K += sneed;
            tokens += sp;
          }
          E += cnt;
          nR += cnt;
          nadm += cnt;
          nrej += nrj;
          adm += stop;
          __syncwarp();
          if (stop < nvalid) break;
        }
      }
    }
    nrej_tot += nrej;
    // 6. empty batch (every candidate rejected): back to 0 without advancing t
    if (nR == 0) continue;
    // block extraction for all requesters of this iteration, in phase order
    if (K > 0 && !alloc_ordered(S, E, K, bt, btl, k, dig_b, hint, nwords)) {
      flags |= TOKENSIM_PT_INTERNAL_ERROR;
      break;
    }
    // 7. cost: decodes are positions [0, D), prefills [D, nR)
    const u32 D = nR3 + (SWAPM ? nres : 0u);
    const u32 Sp = nR - D;
    u64 Np = 0, Ap = 0, Cd = 0;
    for (u32 b0 = 0; b0 < nR; b0 += 32) {
      const u32 jj = b0 + lane;
      if (jj < nR) {
        const u64 c = S.ctx[jj];
        if (jj < D) {
          Cd += c + 1;
        } else {
          Np += c;
          Ap += c * (c + 1) / 2;
        }
      }
    }
    Np = warp_sum64(Np);
    Ap = warp_sum64(Ap);
    Cd = warp_sum64(Cd);
    const i64 T = iter_time_ns(M, H, Np, Ap, Sp, D, Cd, swap_out + swap_in);
    // 8. commit
    const i64 ts = t, te = t + T;
    const u64 blocks = total - nfree;
    u32 nfin = 0, first_fin = 0xffffffffu;
    const u32 fresh0 = nR3 + nres;
    for (u32 b0 = 0; b0 < nR; b0 += 32) {
      const u32 jj = b0 + lane;
      bool fin = false;
      if (jj < nR) {
        const u32 r = S.rem[jj] - 1;
        S.rem[jj] = r;
        if (jj >= fresh0) {
          S.ttft[jj] = te - S.arr[jj];
          S.last[jj] = te;
        } else {
          if (jj < D) S.ctx[jj] += 1;
          const i64 gap = te - S.last[jj];
          if (gap > S.maxgap[jj]) S.maxgap[jj] = gap;
          S.last[jj] = te;
        }
        fin = r == 0;
        if (fin) {
          const u32 id = S.id[jj];
          const i64 ttft = S.ttft[jj], e2e = te - S.arr[jj], mt = S.maxgap[jj];
          const u32 np_ = S.info[jj] >> 16;
          write_record(rec + id, ttft, e2e, mt, np_, TOKENSIM_REQ_FINISHED, (u32)k);
          u64 h = FOLD_INIT;
          h = mix64(h ^ (u64)id);
          h = mix64(h ^ (u64)ttft);
          h = mix64(h ^ (u64)e2e);
          h = mix64(h ^ (u64)mt);
          h = mix64(h ^ (u64)np_);
          h = mix64(h ^ k);
          dig_r += h;
        }
      }
      u32 fm = __ballot_sync(FULLMASK, fin);
      __syncwarp();
      if (fm && first_fin == 0xffffffffu) first_fin = b0 + (u32)(__ffs(fm) - 1);
      nfin += __popc(fm);
      while (fm) {
        const u32 l = (u32)(__ffs(fm) - 1);
        fm &= fm - 1;
        const u32 pos = b0 + l;
        const u32 c = S.ctx[pos];
        const u32 held = (c + bs - 1) / bs;
        const u32 slot = S.info[pos] & 0xffffu;
        free_blocks(S.bitmap, bt + (size_t)slot * btl, held, S.id[pos], k, dig_b, hint);
        nfree += held;
        if (lane == 0) atomicOr(&S.btfree[slot >> 5], 1u << (slot & 31u));
      }
    }
    __syncwarp();
    req_iters += nR;
    if (nfin) {
      // stable compaction of R u Q, dropping finished entries (rem == 0 within R)
      const u32 len = nR + nQ;
      u32 out = first_fin;
      for (u32 b0 = first_fin; b0 < len; b0 += 32) {
        const u32 jj = b0 + lane;
        const bool valid = jj < len;
        u32 vid = 0, vctx = 0, vrem = 0, vinfo = 0;
        i64 vl = 0, vm = 0, va = 0, vt = 0;
        if (valid) {
          vid = S.id[jj];
          vctx = S.ctx[jj];
          vrem = S.rem[jj];
          vinfo = S.info[jj];
          vl = S.last[jj];
          vm = S.maxgap[jj];
          va = S.arr[jj];
          vt = S.ttft[jj];
        }
        const bool keep = valid && vrem != 0;
        const u32 km = __ballot_sync(FULLMASK, keep);
        __syncwarp();
        if (keep) {
          const u32 d = out + __popc(km & ltm);
          S.id[d] = vid;
          S.ctx[d] = vctx;
          S.rem[d] = vrem;
          S.info[d] = vinfo;
          S.last[d] = vl;
          S.maxgap[d] = vm;
          S.arr[d] = va;
          S.ttft[d] = vt;
        }
        __syncwarp();
        out += __popc(km);
      }
      nR -= nfin;
      nfin_tot += nfin;
      last_fin = te;
    }
    // schedule digest fields (buffered; folded 32 iterations at a time)
    if (lane == (u32)(k & 31)) {
      b_k = (u32)k;
      b_t = ts;
      b_T = T;
      b_spd = Sp | (D << 16);
      b_np = Np;
      b_cd = Cd;
      b_mres = m | (nres << 16);
      b_adfin = nadm | (nfin << 16);
      b_rej = nrej;
      b_blk = (u32)blocks;
      b_valid = true;
    }
    if ((k & 31) == 31) flush_sched();
    peak = blocks > peak ? blocks : peak;
    bns += blocks * (u64)T;
    swo_tot += swap_out;
    swi_tot += swap_in;
    if (BINNED) {
      while (bin_end <= ts) flush_bin();
      ++acc_nit;
      i64 s = ts;
      while (te > bin_end) {
        if (bin_end > s) {
          acc_bns += blocks * (u64)(bin_end - s);
          acc_max = max(acc_max, (u32)blocks);
        }
        s = bin_end;
        flush_bin();
      }
      if (te > s) {
        acc_bns += blocks * (u64)(te - s);
        acc_max = max(acc_max, (u32)blocks);
      }
    } else if (FULLT) {
      if (tn < P.trace_cap) {
        if (lane == 0) {
          tokensim_mem_sample s;
          s.t_ns = ts;
          s.dur_ns = T;
          s.block_ns = blocks * (u64)T;
          s.blocks_max = (u32)blocks;
          s.n_iter = 1;
          trc[tn] = s;
        }
      } else {
        flags |= TOKENSIM_PT_TRACE_OVERFLOW;
      }
      ++tn;
    }
    t = te;
    ++k;
  }
  flush_sched();
  if (BINNED) {
    while ((i64)bin * W < t) flush_bin();
  }
  // unfinished requests still in R u Q: first-token latency and preemption count
  for (u32 x = lane; x < nR + nQ; x += 32) {
    const u32 id = S.id[x];
    write_record(rec + id, S.ttft[x], 0, 0, S.info[x] >> 16, TOKENSIM_REQ_UNFINISHED, 0);
  }
  dig_s = warp_sum64(dig_s);
  dig_b = warp_sum64(dig_b);
  dig_r = warp_sum64(dig_r);
  if (lane == 0) {
    SimStats st;
    st.flags = flags | ((nrej_tot == n) ? (u32)TOKENSIM_PT_ALL_REJECTED : 0u);
    st.pad = 0;
    st.n_finished = nfin_tot;
    st.n_rejected = nrej_tot;
    st.n_iterations = k;
    st.n_req_iters = req_iters;
    st.n_preempt = npre;
    st.swap_out = swo_tot;
    st.swap_in = swi_tot;
    st.last_finish = last_fin;
    st.t_final = t;
    st.sched_d = dig_s;
    st.block_d = dig_b;
    st.req_d = dig_r;
    st.total_blocks = total;
    st.peak_blocks = peak;
    st.block_ns_sum = bns;
    st.trace_n[0] = min(tn, P.trace_cap);
    st.trace_n[1] = 0;
    st.iter_n = min(k, P.it_cap);
    st.n_transfers = 0;
    st.transfer_bytes = 0;
    st.reserved[0] = st.reserved[1] = st.reserved[2] = 0;
    P.stats[j] = st;
  }
  __syncwarp();
}

template <int CAP>
__global__ void __launch_bounds__(128) sim_kernel(SweepParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const u32 lane = lane_id(), wib = threadIdx.x >> 5;
  const size_t per_warp = smem_per_warp_bytes(CAP, P.nwords_max);
  const WarpSmem S = carve(smem_raw + wib * per_warp, CAP);
  const u32 gwarp = blockIdx.x * (blockDim.x >> 5) + wib;
  u32 *bt = P.bt + (size_t)gwarp * 2 * CAP * P.bt_len;
  while (true) {
    u32 qi = 0;
    if (lane == 0) qi = atomicAdd(P.queue, 1u);
    qi = __shfl_sync(FULLMASK, qi, 0);
    if ((u64)qi >= P.n_run) break;
    const u64 j = P.order[qi];
    simulate_unified<CAP>(P, j, S, bt);
  }
}

template <int CAP>
static cudaError_t launch_sim_t(const SweepParams &p, int wpb, int blocks, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(sim_kernel<CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  sim_kernel<CAP><<<blocks, wpb * 32, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_sim(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  switch (cap) {
    case 32: return launch_sim_t<32>(p, wpb, blocks, smem, st);
    case 256: return launch_sim_t<256>(p, wpb, blocks, smem, st);
    case 1024: return launch_sim_t<1024>(p, wpb, blocks, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int CAP>
static cudaError_t occ_t(int wpb, size_t smem, int *b) {
  cudaError_t e = cudaFuncSetAttribute(sim_kernel<CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(b, sim_kernel<CAP>, wpb * 32, smem);
}
cudaError_t sim_occupancy(int cap, int wpb, size_t smem, int *b) {
  switch (cap) {
    case 32: return occ_t<32>(wpb, smem, b);
    case 256: return occ_t<256>(wpb, smem, b);
    case 1024: return occ_t<1024>(wpb, smem, b);
    default: return cudaErrorInvalidValue;
  }
}

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
  u64 g_mt = 0, g_both = 0, s_ttft = 0, s_e2e = 0, s_mt = 0;
  for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
    const tokensim_request_record r = rec[i];
    if (r.status != TOKENSIM_REQ_FINISHED) continue;
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
  // sequential fp64 sums for TPOT / NORM in ascending id (SURVEY c.6)
  __shared__ double seq_tp, seq_norm;
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (u32 i = 0; i < n; ++i) {
      const tokensim_request_record r = rec[i];
      if (r.status != TOKENSIM_REQ_FINISHED) continue;
      const u32 o = OU[i];
      if (o >= 2) a = __dadd_rn(a, __ddiv_rn(__ll2double_rn(r.e2e_ns - r.ttft_ns), __uint2double_rn(o - 1)));
      b = __dadd_rn(b, __ddiv_rn(__ll2double_rn(r.e2e_ns), __uint2double_rn(o)));
    }
    seq_tp = a;
    seq_norm = b;
  }
  __syncthreads();
  tokensim_summary S;
  const u64 nfin = st.n_finished;
  const u32 qbp[4] = {5000, 9000, 9900, 10000};
  for (u32 m = 0; m < 5; ++m) {
    u64 kmin, kmax;
    const u32 cnt = build_keys(m, rec, OU, n, keys, sh, kmin, kmax);
    for (u32 qi = 0; qi < 4; ++qi) {
      double v = 0.0;
      if (cnt) {
        const u64 key = qi == 3 ? kmax : block_select(keys, cnt, nearest_rank(qbp[qi], cnt), kmin, kmax, sh);
        v = __longlong_as_double((long long)key);
      }
      S.stat[m][qi] = v;
    }
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
    S.n_requests = n;
    S.n_finished = nfin;
    S.n_rejected = st.n_rejected;
    S.n_unfinished = n - nfin - st.n_rejected;
    S.n_iterations = st.n_iterations;
    S.n_request_iterations = st.n_req_iters;
    S.n_preemptions = st.n_preempt;
    S.swap_out_bytes = st.swap_out;
    S.swap_in_bytes = st.swap_in;
    S.first_arrival_ns = n ? A[0] : 0;
    S.last_finish_ns = st.last_finish;
    S.sched_digest = st.sched_d;
    S.block_digest = st.block_d;
    S.request_digest = st.req_d;
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
