// sim_core.cuh -- a.2-a.7: the persistent per-point simulation kernel.
// Included by sim_base.cu (MIXED unified sweeps: every later feature compiled out, so the
// common path keeps its registers and instruction footprint -- the kernel is instruction-fetch
// bound at 8 warps/SM) and sim_full.cu (prefill-first and chunked iterations, multi-round +
// memory cache, preload link, the P/D pair and the xP:yD node).
//
// ONE WARP PER POINT, pulled from an atomic longest-first queue.  The running set R and
// the resume queue Q are one array of request slots in ascending id (R is a prefix, Q
// the suffix: preemption moves the R/Q boundary left, resume moves it right), held
// structure-of-arrays in shared memory together with the free-block bitmap and the
// block-table slot pool.  Per-slot work is lane-parallel (32 slots per warp step);
// FCFS admission is a prefix scan + ballot; the victim count is the closed form of c.4
// step 3; block allocation extracts the K lowest free bits of the bitmap in one pass
// and hands them out in phase/id order (reading A14).
//
// Quiescent decode stretches are evaluated time-parallel: when no
// admission, resume, preemption or finish can happen for a while, lane j computes
// iteration k+j (its cost, start time by a 64-bit prefix scan, its block allocations,
// its schedule digest and trace sample) and the warp commits up to 32 iterations at
// once -- bit-identical to stepping them one by one.
//
// PAPER.md anchors: worker loop / default end-of-iteration breakpoint P:243; continuous
// vs static batching P:166-169; PagedAttention P:172-173; preemption
// P:456-457; max-memory-ratio admission P:460; compute simulator P:216.
#pragma once
#include "dev_common.cuh"
#include "trace_codec.cuh"

// Latency fast paths that cost more in instruction fetch than they save at 8 warps per SM
// (DESIGN.md §8 A/B log): the fused small-allocation path of a stretch is compiled only into
// the one-warp-per-SM / full kernels.  TS_AB_* switch further ones off for A/B experiments.
#ifndef TS_NO_FUSED
#define TS_NO_FUSED TS_COMPACT
#endif
#ifndef TS_AB_NO_ONEADM
#define TS_AB_NO_ONEADM 0
#endif
#ifndef TS_AB_NO_BTFAST
#define TS_AB_NO_BTFAST 0
#endif
#ifndef TS_AB_NO_HEADQ
#define TS_AB_NO_HEADQ 0
#endif

namespace ts {

// ------------------------------------------------------------------ a.6 cost model
// All F_o/B_o of the c.5 table are integers < 2^53 (validated at create), so forming them
// with fp64 products/sums is exact and equals (double)(u64 value) -- the oracle's form.
struct CostK {
  double h, q2g, hq2g, qh, q, q4, hfu, fu, fh, f, Vh, V, s, att_tok, g2, L, twoL, bar_coef;
  double invF, invB, invH, invT, overhead;
  u32 tp;
  double fetch_s;   // NEXT-2: memory-cache fetch seconds per block
  u32 preload;      // NEXT-4: swap-in through a preload buffer (reading R-N4)
  u64 preload_buf;  // buffer bytes
  u64 Lu;           // layers (chunks of a swap-in)
};

__device__ __forceinline__ CostK make_costk(const DevModel &M, const DevModelF &F, const DevHw &H, u32 link_mode = 0,
                                            u64 preload_buf = 0, double fetch_s = 0.0) {
  CostK K;
  K.fetch_s = fetch_s;
  K.preload = link_mode == TOKENSIM_LINK_PRELOAD ? 1u : 0u;
  K.preload_buf = preload_buf;
  K.Lu = M.L;
  K.h = F.h;
  K.q2g = F.q2g;
  K.hq2g = F.hq2g;
  K.qh = F.qh;
  K.q = F.q;
  K.q4 = F.q4;
  K.hfu = F.hfu;
  K.fu = F.fu;
  K.fh = F.fh;
  K.f = F.f;
  K.Vh = F.Vh;
  K.V = F.V;
  K.s = F.s;
  K.att_tok = F.att_tok;
  K.g2 = F.g2;
  K.L = F.L;
  K.twoL = F.twoL;
  K.bar_coef = H.tp > 1 ? __ull2double_rn(2 * (u64)(H.tp - 1) * M.h * M.s) : 0.0;
  K.invF = H.invF;
  K.invB = H.invB;
  K.invH = H.invH;
  K.invT = H.invT;
  K.overhead = H.overhead;
  K.tp = H.tp;
  return K;
}

__device__ __forceinline__ double roof(double F, double B, const CostK &K) {
  return fmax(__dmul_rn(F, K.invF), __dmul_rn(B, K.invB));
}

// NEXT-4 preload pipeline (reading R-N4), lane 0 only: n chunks, load `a`
// once the previous load is done and a buffer slot is free (chunk i-K taken), the consumer takes
// chunk i at S_i = max(C_{i-1}, P_i) and finishes it `b` later; ring holds S_1..S_n.
static __device__ __noinline__ double preload_pipeline(u64 n, double a, double b, u64 K, double *ring) {
  double Pv = 0.0, Cv = 0.0;
  for (u64 i = 1; i <= n; ++i) {
    double ready = Pv;
    if (i > K) ready = fmax(ready, ring[i - K]);
    Pv = __dadd_rn(ready, a);
    const double Sv = fmax(Cv, Pv);
    ring[i] = Sv;
    Cv = __dadd_rn(Sv, b);
  }
  return Cv;
}

// T_ns of a batch from its exact aggregates; SURVEY c.5 order.  Np = sum of prefill lengths,
// Ap = sum of P*c0 + P(P+1)/2, Kp = sum of c0 + P (keys a prefill reads), Slm = LM-head rows of
// the prefill entries (a non-final chunk samples nothing, reading R-N3b).  With a preload link
// and swap_in > 0 (warp-collective then; `ring` = >= L+1 doubles of scratch) the swap-in
// streams layer by layer through the buffer while the layers compute (reading R-N4).
__device__ __forceinline__ i64 iter_time_chunk_ns(const CostK &K, u64 Np, u64 Ap, u64 Kp, u64 Slm, u64 D,
                                                  u64 Cd, u64 swap_out, u64 swap_in = 0, double *ring = nullptr,
                                                  u64 fetch_blocks = 0) {
  const double N = __ull2double_rn(Np + D), S = __ull2double_rn(Slm + D);
  double tQKV = 0.0, tATTP = 0.0, tATTD = 0.0, tO = 0.0, tUP = 0.0, tDOWN = 0.0, tLM = 0.0;
  const double N2 = __dmul_rn(2.0, N);
  if (Np + D > 0) {
    const double Nh = __dmul_rn(N, K.h);
    tQKV = roof(__dmul_rn(N2, K.hq2g), __dmul_rn(K.s, __dadd_rn(__dadd_rn(K.hq2g, Nh), __dmul_rn(N, K.q2g))), K);
    tO = roof(__dmul_rn(N2, K.qh), __dmul_rn(K.s, __dadd_rn(__dadd_rn(K.qh, __dmul_rn(N, K.q)), Nh)), K);
    tUP = roof(__dmul_rn(N2, K.hfu), __dmul_rn(K.s, __dadd_rn(__dadd_rn(K.hfu, Nh), __dmul_rn(N, K.fu))), K);
    tDOWN = roof(__dmul_rn(N2, K.fh), __dmul_rn(K.s, __dadd_rn(__dadd_rn(K.fh, __dmul_rn(N, K.f)), Nh)), K);
  }
  if (Np > 0) {
    const double Npd = __ull2double_rn(Np);
    tATTP = roof(__dmul_rn(K.q4, __ull2double_rn(Ap)),
                 __dmul_rn(K.s, __dadd_rn(__dmul_rn(Npd, K.att_tok), __dmul_rn(K.g2, __ull2double_rn(Kp)))), K);
  }
  if (D > 0) {
    const double Dd = __ull2double_rn(D), Cdd = __ull2double_rn(Cd);
    tATTD = roof(__dmul_rn(K.q4, Cdd), __dmul_rn(K.s, __dadd_rn(__dmul_rn(Dd, K.att_tok), __dmul_rn(K.g2, Cdd))), K);
  }
  if (Slm + D > 0)
    tLM = roof(__dmul_rn(__dmul_rn(2.0, S), K.Vh),
               __dmul_rn(K.s, __dadd_rn(__dadd_rn(K.Vh, __dmul_rn(S, K.h)), __dmul_rn(S, K.V))), K);
  const double tl =
      __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(tQKV, tATTP), tATTD), tO), tUP), tDOWN);
  const bool pipe = K.preload && swap_in > 0;
  double T;
  if (pipe) {
    const u64 chunk = swap_in / K.Lu;  // exact: kvb has a factor L
    const u64 q = K.preload_buf / chunk;
    double c = 0.0;
    if (lane_id() == 0)
      c = preload_pipeline(K.Lu, __dmul_rn(__ull2double_rn(chunk), K.invH), tl, q ? q : 1ull, ring);
    T = __shfl_sync(FULLMASK, c, 0);
  } else {
    T = __dmul_rn(tl, K.L);
  }
  T = __dadd_rn(T, tLM);
  if (K.tp > 1) T = __dadd_rn(T, __dmul_rn(__dmul_rn(__dmul_rn(K.bar_coef, N), K.invT), K.twoL));
  const u64 swap_bytes = pipe ? swap_out : swap_out + swap_in;
  if (swap_bytes > 0) T = __dadd_rn(T, __dmul_rn(__ull2double_rn(swap_bytes), K.invH));
  if (fetch_blocks > 0) T = __dadd_rn(T, __dmul_rn(__ull2double_rn(fetch_blocks), K.fetch_s));  // NEXT-2
  T = __dadd_rn(T, K.overhead);
  return (i64)floor(__dadd_rn(__dmul_rn(T, 1e9), 0.5));
}
// whole prefills (c0 = 0, so K_p = N_p, every entry emits)
__device__ __forceinline__ i64 iter_time_ns(const CostK &K, u64 Np, u64 Ap, u64 Sp, u64 D, u64 Cd,
                                            u64 swap_bytes) {
  return iter_time_chunk_ns(K, Np, Ap, Np, Sp, D, Cd, swap_bytes);
}

// ------------------------------------------------------------------ per-warp shared memory
struct WarpSmem {
  u32 *id, *ctx, *rem, *info;       // info: bt slot (bits 0-15) | n_preempt (bits 16-31)
  i64 *last, *maxgap, *arr, *ttft;  // last token time, max gap, arrival, ttft
  u32 *req_cum, *req_pt;            // block requesters: cumulative count; pos|j<<10|tpos<<15
  u32 *scratch;                     // 64 words: fast-forward histogram / cursors, residue masks
  u32 *btfree;                      // cap/32 words, bit = free block-table slot
  u32 *bitmap;                      // free-block bitmap, bit = free block
};

__host__ __device__ inline size_t smem_per_warp_bytes(u32 cap, u32 nwords_max) {
  size_t b = (size_t)cap * (4 * 4 + 8 * 4 + 4 * 2) + 64 * 4 + (size_t)(cap / 32) * 4 + (size_t)nwords_max * 4;
  return (b + 15) & ~(size_t)15;
}
// P/D extra per warp: slot states, the prefill batch (id, slot, p, o) and P's bitmap
__host__ __device__ inline size_t smem_pd_extra(u32 cap, u32 nwords_max) {
  return ((size_t)cap * 4 * 5 + (size_t)nwords_max * 4 + 15) & ~(size_t)15;
}
size_t sim_smem_per_warp(int cap, u32 nwords_max, bool pd, u32 node_x, u32 node_y);

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
  S.scratch = p32 + 6 * cap;
  S.btfree = p32 + 6 * cap + 64;
  S.bitmap = p32 + 6 * cap + 64 + cap / 32;
  return S;
}

#define PT_POS(pt) ((pt)&1023u)
// info word of a slot: block-table slot (bits 0-9) | CHUNKED flags (bits 14-15) | n_preempt << 16
#define SLOT(info) ((info)&1023u)
constexpr u32 INFO_NT = 1u << 14;   // CHUNKED: no token emitted yet (the next prefill completion is the first token)
constexpr u32 INFO_PFB = 1u << 15;  // CHUNKED: a resumed re-prefill in this iteration's batch
#define PT_J(pt) (((pt) >> 10) & 31u)
#define PT_TPOS(pt) ((pt) >> 15)

// ------------------------------------------------------------------ digest logs
// Digest terms are not folded on the per-iteration dependency chain: block events and
// per-iteration schedule fields are appended to small per-warp logs in global memory and
// folded lane-parallel when a log fills (the digests are wrapping sums: order-free).
constexpr u32 EVCAP = 1024;  // block events per flush
constexpr u32 ITCAP = 256;   // iterations per flush
struct Logs {
  uint4 *ev;
  ulonglong2 *it;               // 4 x 16 B per iteration entry
  tokensim_iter_record *itr;
  u64 it_cap, it_base;          // processing-order index of it[0]
  u64 dig_s, dig_b;             // per-lane partial sums
  u32 nev, nit;
};

// The folds are out of line.  In the lean variant they take/return values, so the Logs fields
// stay in registers (a reference to a local struct puts it on the stack for every append); the
// full variant (sim_full.cu sets TS_LOGS_BYREF) keeps the by-reference form, which measured
// faster there because the stack copy relieves its register pressure.
#if TS_LOGS_BYREF
static __device__ __noinline__ void ev_flush(Logs &L) {
  __syncwarp();
  #pragma unroll 1
  for (u32 x = lane_id(); x < L.nev; x += 32) {
    const uint4 e = L.ev[x];
    L.dig_b += fold_event(e.x, e.y, e.z, e.w);
  }
  L.nev = 0;
  __syncwarp();
}
#else
static __device__ __noinline__ u64 ev_fold(const uint4 *ev, u32 nev) {
  __syncwarp();
  u64 d = 0;
  #pragma unroll 1
  for (u32 x = lane_id(); x < nev; x += 32) {
    const uint4 e = ev[x];
    d += fold_event(e.x, e.y, e.z, e.w);
  }
  __syncwarp();
  return d;
}
__device__ __forceinline__ void ev_flush(Logs &L) {
  L.dig_b += ev_fold(L.ev, L.nev);
  L.nev = 0;
}
#endif
__device__ __forceinline__ void ev_reserve(Logs &L, u32 cnt) {
  if (L.nev + cnt > EVCAP) ev_flush(L);
}
__device__ __forceinline__ void ev_put(Logs &L, u32 idx, u64 k, u32 kind, u32 id, u32 blk) {
  L.ev[L.nev + idx] = make_uint4((u32)k, kind, id, blk);
}

// ------------------------------------------------------------------ a.5 allocator
// Return `held` blocks of table `tbl` to the bitmap (order-free: the block digest is a
// wrapping sum) and lower the lowest-free-word hint.
__device__ __forceinline__ void free_blocks(u32 *bitmap, const u32 *tbl, u32 held, u32 id, u64 k, u32 kind_off,
                                            Logs &L, u32 &hint) {
  u32 mn = 0xffffffffu;
  #pragma unroll 1
  for (u32 x0 = 0; x0 < held; x0 += 32) {
    ev_reserve(L, 32);
    const u32 x = x0 + lane_id();
    if (x < held) {
      const u32 b = tbl[x];
      atomicOr(&bitmap[b >> 5], 1u << (b & 31u));
      ev_put(L, x - x0, k, 2 + kind_off, id, b);
      mn = min(mn, b >> 5);
    }
    L.nev += min(32u, held - x0);
  }
  mn = __reduce_min_sync(FULLMASK, mn);
  hint = min(hint, mn);
}

// Take the K lowest free blocks (in ascending order) into out[0..K) and clear them (32-word
// windows from the hint).  false if fewer than K are free at or above the hint.
static __device__ bool take_lowest(u32 *bitmap, u32 K, u32 *out, u32 &hint, u32 nwords) {
  const u32 lane = lane_id();
  u32 o_base = 0, w = hint;
  while (o_base < K) {
    if (w >= nwords) return false;
    const u32 wi = w + lane;
    u32 word = wi < nwords ? bitmap[wi] : 0u;
    const u32 c = __popc(word);
    const u32 cum = scan_incl(c);
    const u32 tot = __shfl_sync(FULLMASK, cum, 31);
    if (tot == 0) {
      w += 32;
      continue;
    }
    const u32 take = min(tot, K - o_base);
    const u32 before = cum - c;
    #pragma unroll 1
    for (u32 r0 = 0; r0 < take; r0 += 32) {
      const u32 idx = r0 + lane;
      const u32 tgt = idx < take ? idx : 0u;
      u32 lo = 0;
#pragma unroll
      for (u32 s = 16; s; s >>= 1) {
        const u32 v = __shfl_sync(FULLMASK, cum, lo + s - 1);
        if (v <= tgt) lo += s;
      }
      const u32 wv = __shfl_sync(FULLMASK, word, lo);
      const u32 bv = __shfl_sync(FULLMASK, before, lo);
      if (idx < take) out[o_base + idx] = (w + lo) * 32 + select_bit(wv, tgt - bv);
    }
    const u32 tk = take > before ? min(c, take - before) : 0u;
    if (tk && wi < nwords) {
      word = clear_lowest(word, tk, c);
      bitmap[wi] = word;
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

// Hand out the K lowest free blocks, in order, to the E requesters in S.req_* (entry e
// owns order indices [req_cum[e-1], req_cum[e]) and writes its table from tpos).  This is
// "serve the requesters one after another with take-the-lowest-free-block" (c.4 steps
// 3-5, reading A14) done in one bitmap pass.  Entry iteration offsets (fast-forward)
// shift the digest's iteration index.  The first E1 entries take one block each (decode
// requesters come first in phase order), so their owner needs no search.
static __device__ bool alloc_ordered(const WarpSmem &S, u32 E, u32 K, u32 *bt, u32 btl, u64 k, u32 kind_off, Logs &L,
                              u32 &hint, u32 nwords, u32 E1 = 0) {
  if (E == K) E1 = E;  // every requester takes one block: owner of order index o is o
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
    #pragma unroll 1
    for (u32 r0 = 0; r0 < take; r0 += 32) {
      ev_reserve(L, 32);
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
        u32 a = o, start = o;
        if (o >= E1) {
          a = E1;
          u32 bnd = E;
          while (a < bnd) {
            const u32 mid = (a + bnd) >> 1;
            if (S.req_cum[mid] <= o) a = mid + 1;
            else bnd = mid;
          }
          start = a ? S.req_cum[a - 1] : 0u;
        }
        const u32 pt = S.req_pt[a];
        const u32 pos = PT_POS(pt);
        const u32 tpos = PT_TPOS(pt) + (o - start);
        const u32 slot = SLOT(S.info[pos]);
        bt[(size_t)slot * btl + tpos] = blk;
        ev_put(L, idx - r0, k + PT_J(pt), 1 + kind_off, S.id[pos], blk);
      }
      L.nev += min(32u, take - r0);
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
  if (!TS_AB_NO_BTFAST && cnt == 1) {  // one admission (the common case): the lowest set bit of the first nonzero word
    const u32 nz = __ballot_sync(FULLMASK, word != 0u);
    const u32 l = (u32)(__ffs(nz) - 1);
    const u32 wv = __shfl_sync(FULLMASK, word, l);
    if (lane == l) btfree[l] = wv & (wv - 1u);
    __syncwarp();
    return l * 32 + (u32)(__ffs(wv) - 1);
  }
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

// iteration digest term: fold(k | worker << 40, t, T, N_p, C_d, blocks,
//                            S_p | D << 16 | m << 32 | n_res << 48, n_adm | n_fin << 16 | n_rej << 32)
__device__ __forceinline__ u64 sched_fold(u64 k, i64 ts, i64 T, u64 Np, u64 Cd, u64 blocks, u64 w6, u64 w7) {
  u64 h = FOLD_INIT;
  h = mix64(h ^ k);
  h = mix64(h ^ (u64)ts);
  h = mix64(h ^ (u64)T);
  h = mix64(h ^ Np);
  h = mix64(h ^ Cd);
  h = mix64(h ^ blocks);
  h = mix64(h ^ w6);
  h = mix64(h ^ w7);
  return h;
}

// iteration entry: k (worker in bit 40), t_start, T, N_p, C_d, blocks,
// S_p | D<<16 | m<<32 | n_resumed<<48, n_admitted | n_finished<<16 | n_rejected<<32
static __device__ __noinline__ u64 it_fold(const ulonglong2 *it, u32 nit, tokensim_iter_record *itr, u64 it_cap,
                                          u64 it_base) {
  __syncwarp();
  u64 dg = 0;
  #pragma unroll 1
  for (u32 x = lane_id(); x < nit; x += 32) {
    const ulonglong2 a = it[4 * x], b = it[4 * x + 1], c = it[4 * x + 2], d = it[4 * x + 3];
    const u64 k = a.x, Np = b.y, Cd = c.x, blocks = c.y, w6 = d.x, w7 = d.y;
    const i64 ts = (i64)a.y, T = (i64)b.x;
    const u64 Sp = w6 & 0xffff, D = (w6 >> 16) & 0xffff, m = (w6 >> 32) & 0xffff, nres = w6 >> 48;
    const u64 nadm = w7 & 0xffff, nfin = (w7 >> 16) & 0xffff, nrej = w7 >> 32;
    dg += sched_fold(k, ts, T, Np, Cd, blocks, w6, w7);
    const u64 idx = it_base + x;
    if (idx < it_cap) {
      tokensim_iter_record ir;
      ir.k = k & ((1ull << 40) - 1);
      ir.t_start_ns = ts;
      ir.T_ns = T;
      ir.n_prefill = (u32)Sp;
      ir.n_decode = (u32)D;
      ir.N_p = Np;
      ir.C_d = Cd;
      ir.n_preempted = (u32)m;
      ir.n_resumed = (u32)nres;
      ir.n_admitted = (u32)nadm;
      ir.n_rejected = (u32)nrej;
      ir.n_finished = (u32)nfin;
      ir.blocks_in_use = (u32)blocks;
      ir.worker = (u32)(k >> 40);
      ir.pad = 0;
      itr[idx] = ir;
    }
  }
  __syncwarp();
  return dg;
}
#if TS_LOGS_BYREF
static __device__ __noinline__ void it_flush(Logs &L) {
  L.dig_s += it_fold(L.it, L.nit, L.itr, L.it_cap, L.it_base);
  L.it_base += L.nit;
  L.nit = 0;
}
#else
__device__ __forceinline__ void it_flush(Logs &L) {
  L.dig_s += it_fold(L.it, L.nit, L.itr, L.it_cap, L.it_base);
  L.it_base += L.nit;
  L.nit = 0;
}
#endif
__device__ __forceinline__ void it_reserve(Logs &L, u32 cnt) {
  if (L.nit + cnt > ITCAP) it_flush(L);
}
__device__ __forceinline__ void it_put(Logs &L, u32 idx, u64 k, i64 ts, i64 T, u64 Np, u64 Cd, u64 blocks, u64 Sp,
                                       u64 D, u64 m, u64 nres, u64 nadm, u64 nfin, u64 nrej) {
  ulonglong2 *e = L.it + 4 * (size_t)((L.nit + idx) & (ITCAP - 1));  // a ring in helper mode
  e[0] = make_ulonglong2(k, (unsigned long long)ts);
  e[1] = make_ulonglong2((unsigned long long)T, Np);
  e[2] = make_ulonglong2(Cd, blocks);
  e[3] = make_ulonglong2(Sp | (D << 16) | (m << 32) | (nres << 48), nadm | (nfin << 16) | (nrej << 32));
}

TS_SCANFN i64 scan_incl_i64(i64 x) {
  const u32 l = lane_id();
#pragma unroll
  for (u32 o = 1; o < 32; o <<= 1) {
    const i64 y = __shfl_up_sync(FULLMASK, x, o);
    if (l >= o) x += y;
  }
  return x;
}

#include "sim_pd.cuh"
#include "sim_pdn.cuh"

// per simulated point: a warp's worth, or a whole node CTA's
inline size_t sim_smem_per_warp_impl(int cap, u32 nwords_max, bool pd, u32 node_x, u32 node_y) {
  if (node_x) return pdn_smem_per_warp((u32)cap, nwords_max, node_x, node_y);
  return smem_per_warp_bytes((u32)cap, nwords_max) + (pd ? smem_pd_extra((u32)cap, nwords_max) : 0);
}

// ------------------------------------------------------------------ NEXT-2 per-point state
// Multi-round conversations and the host memory cache (reading R-N2).  All of this is scalar
// code run identically by every lane (equal values written to equal addresses), so the state
// stays lane-uniform without broadcasts.
constexpr u32 MR_NIL = 0xffffffffu;
struct MrState {
  const u32 *CONV, *BASE, *NR;
  u32 *wq_id;          // arrival FIFO: request ids in arrival order, and their arrival times
  i64 *wq_t;
  i64 *hp_t;           // follow-up rounds: min-heap on (time, conversation)
  u32 *hp_c;
  u32 *nxr;            // round index of a conversation's pending follow-up
  u32 *ctok;           // cached context tokens per conversation (0 = not cached)
  u32 *lprev, *lnext;  // LRU list (head = least recently used)
  u32 nconv, ntot, next0, hsize, lhead, ltail;
  u64 used, cap;
};
__device__ __forceinline__ bool mr_less(i64 t1, u32 c1, i64 t2, u32 c2) { return t1 < t2 || (t1 == t2 && c1 < c2); }
__device__ __forceinline__ void mr_heap_push(MrState &M, i64 t, u32 c) {
  u32 i = M.hsize++;
  while (i > 0) {
    const u32 p = (i - 1) >> 1;
    if (!mr_less(t, c, M.hp_t[p], M.hp_c[p])) break;
    M.hp_t[i] = M.hp_t[p];
    M.hp_c[i] = M.hp_c[p];
    i = p;
  }
  M.hp_t[i] = t;
  M.hp_c[i] = c;
}
__device__ __forceinline__ void mr_heap_pop(MrState &M) {
  const u32 n = --M.hsize;
  if (n == 0) return;
  const i64 t = M.hp_t[n];
  const u32 c = M.hp_c[n];
  u32 i = 0;
  while (true) {
    u32 l = 2 * i + 1;
    if (l >= n) break;
    if (l + 1 < n && mr_less(M.hp_t[l + 1], M.hp_c[l + 1], M.hp_t[l], M.hp_c[l])) ++l;
    if (!mr_less(M.hp_t[l], M.hp_c[l], t, c)) break;
    M.hp_t[i] = M.hp_t[l];
    M.hp_c[i] = M.hp_c[l];
    i = l;
  }
  M.hp_t[i] = t;
  M.hp_c[i] = c;
}
// the next arrival (round 0 stream vs pending follow-ups), ties to the lower conversation
__device__ __forceinline__ bool mr_next(const MrState &M, const i64 *A, i64 &ta, u32 &cv, bool &from0) {
  ta = INT64_MAX;
  from0 = false;
  bool any = false;
  if (M.next0 < M.nconv) {
    ta = A[M.BASE[M.next0]];
    cv = M.next0;
    from0 = true;
    any = true;
  }
  if (M.hsize) {
    const i64 ht = M.hp_t[0];
    const u32 hc = M.hp_c[0];
    if (!any || mr_less(ht, hc, ta, cv)) {
      ta = ht;
      cv = hc;
      from0 = false;
      any = true;
    }
  }
  return any;
}
__device__ __forceinline__ void mr_unlink(MrState &M, u32 c) {
  const u32 p = M.lprev[c], nx = M.lnext[c];
  if (p != MR_NIL) M.lnext[p] = nx;
  else M.lhead = nx;
  if (nx != MR_NIL) M.lprev[nx] = p;
  else M.ltail = p;
}
__device__ __forceinline__ void mr_append(MrState &M, u32 c) {
  M.lprev[c] = M.ltail;
  M.lnext[c] = MR_NIL;
  if (M.ltail != MR_NIL) M.lnext[M.ltail] = c;
  else M.lhead = c;
  M.ltail = c;
}
// a finishing round stores its context as the most recently used entry; evict LRU entries
__device__ __forceinline__ void mr_cache_store(MrState &M, u32 c, u32 tokens, const BSz &B) {
  if (M.ctok[c]) {
    M.used -= B.cdiv(M.ctok[c]);
    mr_unlink(M, c);
    M.ctok[c] = 0;
  }
  const u64 blk = B.cdiv(tokens);
  if (blk > M.cap) return;  // larger than the whole cache
  mr_append(M, c);
  M.ctok[c] = tokens;
  M.used += blk;
  while (M.used > M.cap) {
    const u32 e = M.lhead;
    mr_unlink(M, e);
    M.used -= B.cdiv(M.ctok[e]);
    M.ctok[e] = 0;
  }
}

// ------------------------------------------------------------------ a.2-a.7 one point
// Everything is executed by all 32 lanes; scalar state is lane-uniform in registers.
// ------------------------------------------------------------------ helper warp (TS_HELPER_WARP)
// In the one-warp-per-SM lean kernel (sim_base.cu) a second warp of the CTA consumes the
// iteration log: schedule digest, iteration records, memory trace, block-ns sum and peak are
// all functions of the logged (k, t, T, N_p, C_d, blocks, ...) entries, so they leave the
// simulating warp's serial chain.  The log is a 256-entry ring in global memory; the two warps
// hand over through counters in shared memory.  Every wait is bounded (~10 s of clock) and
// raises TOKENSIM_PT_INTERNAL_ERROR instead of hanging.
#ifndef TS_SPEC  // A/B: the second stretch half's costs evaluated alongside the first
#define TS_SPEC 0
#endif
#ifndef TS_XS  // the helper kernel's extended stretches (0: sim_base_n.cu, for several points per SM)
#define TS_XS 1
#endif
#ifndef TS_HELPER_WARP
#define TS_HELPER_WARP 0
#endif
struct HelperChan {
  u32 state;  // 0 idle, 1 point running, 2 simulation done, 3 helper done, 4 exit
  u32 prod, cons, tflags;   // iteration-log ring
  u32 eprod, econs, pad0, pad1;  // block-event ring (allocations / frees to replay)
  u64 j;
  i64 t_final;
  u64 dig, bns, peak, tn, digb, tb;  // tb: FULL trace bytes (trace_codec.cuh)
};
// Block-event records of the helper mode (uint4): k, kind | count << 2, request id,
// table slot | table position << 10.  kind 1: take `count` lowest free blocks into the slot's
// table from the position; kind 2: return the slot's first `count` blocks.
constexpr u32 HEV_ALLOC = 1, HEV_FREE = 2;
constexpr long long HELPER_TIMEOUT = 20000000000ll;  // cycles
__device__ __forceinline__ u32 chan_load(const volatile u32 *p) { return __shfl_sync(FULLMASK, *p, 0); }

// Replay block events [econs, eprod) of a warp's event ring on a bitmap, in order (a.5,
// reading A14: lowest free block first, frees in logical order): allocations write the block
// tables and fold the block digest, frees return a table's first `count` blocks.  Consecutive
// allocations are served by one extraction.  Used by the helper warp (one point per SM) and by
// the several-warps-per-SM lean kernel, whose simulating warp drains its own ring when it fills
// (the simulation itself needs block counts only).  false: the bitmap ran out (an internal error).
static __device__ __noinline__ bool replay_block_events(const uint4 *evr, u32 &econs, u32 eprod, u32 *hbm, u32 *fl,
                                                        u32 &hint, u32 nwords, u32 *bt, u32 btl, u64 &dgb) {
  const u32 lane = lane_id();
  bool ev_err = false;
  #pragma unroll 1
  while (econs != eprod) {  // block events, in order
    const u32 m = min(32u, eprod - econs);
    const bool v = lane < m;
    uint4 ev = make_uint4(0, 0, 0, 0);
    if (v) ev = evr[(econs + lane) & (EVCAP - 1)];
    const u32 kind = ev.y & 3u, cnt = ev.y >> 2;
    const u32 fm = __ballot_sync(FULLMASK, v && kind == HEV_FREE);
    if (fm & 1u) {  // a free: return the slot's first cnt blocks
      const u32 kk = __shfl_sync(FULLMASK, ev.x, 0), held = __shfl_sync(FULLMASK, cnt, 0);
      const u32 id = __shfl_sync(FULLMASK, ev.z, 0), slot = __shfl_sync(FULLMASK, ev.w, 0) & 1023u;
      u32 mn = 0xffffffffu;
      #pragma unroll 1
      for (u32 x = lane; x < held; x += 32) {
        const u32 b = bt[(size_t)slot * btl + x];
        atomicOr(&hbm[b >> 5], 1u << (b & 31u));
        dgb += fold_event(kk, 2, id, b);
        mn = min(mn, b >> 5);
      }
      mn = __reduce_min_sync(FULLMASK, mn);
      hint = min(hint, mn);
      __syncwarp();
      econs += 1;
      continue;
    }
    const u32 na = fm ? (u32)(__ffs(fm) - 1) : m;  // leading allocations
    const u32 c = lane < na ? cnt : 0u;
    const u32 cum = scan_incl(c);
    const u32 K = __shfl_sync(FULLMASK, cum, na - 1);
    if (K <= 256) {  // all of them from one extraction, lane per block
      if (K && !take_lowest(hbm, K, fl, hint, nwords)) ev_err = true;
      #pragma unroll 1
      for (u32 o0 = 0; o0 < K; o0 += 32) {
        const u32 o = o0 + lane;
        const u32 tgt = o < K ? o : 0u;
        u32 a = 0;
#pragma unroll
        for (u32 st = 16; st; st >>= 1) {
          const u32 vv = __shfl_sync(FULLMASK, cum, a + st - 1);
          if (vv <= tgt) a += st;
        }
        const u32 ex = __shfl_sync(FULLMASK, cum - c, a);
        const u32 kk = __shfl_sync(FULLMASK, ev.x, a), id = __shfl_sync(FULLMASK, ev.z, a);
        const u32 sw = __shfl_sync(FULLMASK, ev.w, a);
        if (o < K) {
          const u32 blk = fl[o];
          bt[(size_t)(sw & 1023u) * btl + (sw >> 10) + (o - ex)] = blk;
          dgb += fold_event(kk, 1, id, blk);
        }
      }
      __syncwarp();
    } else {  // a large request: event by event, 256 blocks at a time
      #pragma unroll 1
      for (u32 i = 0; i < na; ++i) {
        const u32 kk = __shfl_sync(FULLMASK, ev.x, i), id = __shfl_sync(FULLMASK, ev.z, i);
        const u32 sw = __shfl_sync(FULLMASK, ev.w, i), ci = __shfl_sync(FULLMASK, cnt, i);
        #pragma unroll 1
        for (u32 s0 = 0; s0 < ci; s0 += 256) {
          const u32 kc = min(256u, ci - s0);
          if (!take_lowest(hbm, kc, fl, hint, nwords)) ev_err = true;
          #pragma unroll 1
          for (u32 x = lane; x < kc; x += 32) {
            const u32 blk = fl[x];
            bt[(size_t)(sw & 1023u) * btl + (sw >> 10) + s0 + x] = blk;
            dgb += fold_event(kk, 1, id, blk);
          }
          __syncwarp();
        }
      }
    }
    econs += na;
  }
  return !ev_err;
}


template <int CAP, bool FULL, bool P2>
__device__ void simulate_unified(const SweepParams &P, u64 j, const WarpSmem &S, u32 *bt,
                                 volatile HelperChan *ch = nullptr) {
  constexpr bool HELP = TS_HELPER_WARP;  // V 0 / 5 (lean) and V 6 (full) are built with the helper warp
  // Extended stretches (carried stretch state, up to 64 iterations per stretch) only in the
  // latency-bound helper-warp kernel: they shorten a lone point's chain, but at 8 warps per SM
  // the larger hot code costs more in instruction fetch than it saves (DESIGN.md §8 A/B log).
  constexpr bool XS = HELP && TS_XS;
  // Block ids off the simulation chain (HEV): every scheduling decision depends on block counts
  // only, so allocations and frees are logged as events in a per-warp ring and the helper warp
  // replays the ring into block ids (tables, bitmap, block digest).  The several-warps-per-SM
  // kernel replaying its own ring whenever it fills (SD) was measured: bit-identical, but C3
  // 614 -> 668 ms, so it keeps its inline allocator.
  constexpr bool SD = false;
  constexpr bool HEV = HELP || SD;
  static_assert(CAP % 32 == 0 && CAP <= 1024, "CAP");
  const u32 lane = lane_id();
  const u32 ltm = lanemask_lt();
  const u64 point = P.begin + j * P.stride;
  const Coords cd = decode_point(point, P.n_pol, P.n_rates, P.n_seeds);
  const DevHw H = P.hw[cd.hw];
  const DevHP HP = P.hp[(size_t)cd.hw * P.n_pol + cd.pol];
  const DevPol PL = P.pol[cd.pol];
  const CostK K = make_costk(P.M, P.MF, H, FULL ? P.link_mode : 0u, P.preload_buf, FULL ? P.fetch_s : 0.0);
  const u32 g = P.group_of_point_mode ? 0u : cd.rate * P.n_seeds + cd.seed;
  const u32 n = P.n_req;
  const i64 *A = P.arrival + (size_t)g * n;
  const u32 *PR = P.prompt + (size_t)g * n;
  const u32 *OU = P.output + (size_t)g * n;
  tokensim_request_record *rec = P.rec + (size_t)j * n;
  tokensim_mem_sample *trc = P.trace + (size_t)j * P.trace_nw * P.trace_cap;
  tokensim_iter_record *itr = P.itrec + (size_t)j * P.it_cap;
  const BSz B = {PL.bs, PL.bs_sh, PL.bs - 1u, P2 || PL.bs_sh != 0xffffffffu};  // P2: folded to shifts
  const bool SWAPM = PL.preempt == TOKENSIM_SWAP;
  const bool RATIO = PL.kind == TOKENSIM_CONT_RATIO;
  const bool STATICP = PL.kind == TOKENSIM_STATIC;
  const bool PFM = FULL && PL.mode == TOKENSIM_PREFILL_FIRST;  // the lean variant runs MIXED only
  const bool CHK = FULL && PL.mode == TOKENSIM_CHUNKED;
  const bool MRM = FULL && P.multi_round != 0;  // NEXT-2: request ids are (conversation, round) rids
  const bool CACHE = MRM && P.memory_cache != 0;
  const u64 total = HP.total_blocks;
  const u32 nwords = HP.nwords;
  const u32 btl = P.bt_len;
  const u32 mns = PL.mns, mbt = PL.mbt;
  const i64 wm = (i64)PL.wm;
  const bool ff_on = P.ff_enable != 0;
  const long long clk0 = clock64();

  // ---- init: records, bitmap, slot pool
  {
    ulonglong2 *r2 = reinterpret_cast<ulonglong2 *>(rec);
    const ulonglong2 z = make_ulonglong2(0ull, 0ull);
    #pragma unroll 1
    for (u32 x = lane; x < 2 * n; x += 32) r2[x] = z;
    const u32 full_words = (u32)(total >> 5), tail = (u32)(total & 31u);
    #pragma unroll 1
    for (u32 w = lane; w < nwords; w += 32)
      S.bitmap[w] = w < full_words ? 0xffffffffu : (w == full_words && tail ? ((1u << tail) - 1u) : 0u);
    #pragma unroll 1
    for (u32 w = lane; w < CAP / 32; w += 32) S.btfree[w] = 0xffffffffu;
    __syncwarp();
  }

  i64 t = 0;
  u64 k = 0;
  u32 arr = 0, adm = 0, nR = 0, nQ = 0;
  u64 nfree = total;
  u32 hint = 0;
  u32 rmin = 0;  // min rem over R after the last commit (0 when unknown / R empty)
  // Stretch state carried from one stretch to the next (valid only between back-to-back
  // stretches; any normal iteration clears it): C_d = sum(ctx + 1) over R and, on lane r < bs,
  // the number of running slots whose next block boundary is r iterations ahead (j0 = -ctx mod
  // bs).  A stretch of J iterations rotates that histogram by J and drops its finished slots, so
  // the next stretch starts without a pass over R (block sizes <= 32 only).
  bool inc_ok = false;
  u64 inc_cd = 0;
  u32 inc_h = 0;  // lane r: running slots of residue class r
  // CHUNKED (NEXT-3b): the budget runs out at the last prefill entry of an iteration, so at most
  // one prefill is in progress and it is the last entry of R (reading R-N3b): xdone of xtgt done
  bool hx = false;
  u32 xdone = 0, xtgt = 0;
  u64 ff_mem_wait = 0, ff_mem_k = 0;  // after a memory-cut failure: skip attempts while nfree <= wait, k < k
  const u32 gwarp = HELP ? blockIdx.x : blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  Logs L;
  L.ev = P.evlog + (size_t)gwarp * EVCAP;
  L.it = P.itlog + (size_t)gwarp * ITCAP * 4;
  L.itr = itr;
  L.it_cap = P.it_cap;
  L.it_base = 0;
  L.dig_s = 0;
  L.dig_b = 0;
  L.nev = 0;
  L.nit = 0;
  u32 flags = 0;
  // the helper's consumer counters as last seen: they only grow, so a stale copy is a safe
  // (pessimistic) bound and the shared-memory load + broadcast is paid only when it says full
  u32 cons_seen = 0, econs_seen = 0;
  // iteration-log hand-over: reserve cnt entries / publish the entries written
  auto it_begin = [&](u32 cnt) {
    if constexpr (HELP) {
      if (L.nit + cnt - cons_seen <= ITCAP) return;
      const long long c0 = clock64();
      while (L.nit + cnt - (cons_seen = chan_load(&ch->cons)) > ITCAP) {
        if (clock64() - c0 > HELPER_TIMEOUT) {
          flags |= TOKENSIM_PT_INTERNAL_ERROR;
          break;
        }
      }
    } else {
      it_reserve(L, cnt);
    }
  };
  // one fence per iteration publishes both rings (iteration entries and block events)
  auto it_commit = [&]() {
    if constexpr (HELP) {
      __threadfence_block();
      __syncwarp();
      if (lane_id() == 0) {
        ch->eprod = L.nev;
        ch->prod = L.nit;
      }
    }
  };
  // helper mode: block ids are output-only (every decision uses counts), so allocations and
  // frees are logged as events and replayed on the bitmap by the helper warp
  auto ev_commit = [&]() {
    __threadfence_block();
    __syncwarp();
    if (lane_id() == 0) ch->eprod = L.nev;
  };
  u64 sd_dgb = 0;  // SD: block-digest partial of this lane (replay_block_events)
  auto sd_drain = [&]() {  // SD: replay every logged block event (on this warp's bitmap)
    __syncwarp();
    if (!replay_block_events(L.ev, econs_seen, L.nev, S.bitmap, S.req_cum, hint, nwords, bt, btl, sd_dgb))
      flags |= TOKENSIM_PT_INTERNAL_ERROR;
  };
  auto ev_begin = [&](u32 cnt) {  // room for cnt events; publish first if we must wait
    if (L.nev + cnt - econs_seen <= EVCAP) return;
    if constexpr (SD) {
      sd_drain();
      return;
    }
    if (L.nev + cnt - (econs_seen = chan_load(&ch->econs)) <= EVCAP) return;
    ev_commit();
    const long long c0 = clock64();
    while (L.nev + cnt - (econs_seen = chan_load(&ch->econs)) > EVCAP) {
      if (clock64() - c0 > HELPER_TIMEOUT) {
        flags |= TOKENSIM_PT_INTERNAL_ERROR;
        break;
      }
    }
  };
  auto ev_log = [&](u32 idx, u64 kk, u32 kind, u32 count, u32 id, u32 slot, u32 tpos) {
    L.ev[(L.nev + idx) & (EVCAP - 1)] = make_uint4((u32)kk, kind | (count << 2), id, slot | (tpos << 10));
  };
  // free (kind 2) of a request's `held` blocks: one event from lane 0
  auto ev_free = [&](u32 held, u32 id, u32 slot, u64 kk) {
    ev_begin(1);
    if (lane_id() == 0) ev_log(0, kk, HEV_FREE, held, id, slot, 0);
    L.nev += 1;
  };
  MrState mr;
  if (MRM) {
    unsigned char *mb = P.mr_scratch + (size_t)gwarp * P.mr_bytes_per_warp;
    const u32 nc = P.n_conv;
    mr.CONV = P.mr_conv + (size_t)g * n;
    mr.BASE = P.mr_base + (size_t)g * nc;
    mr.NR = P.mr_nr + (size_t)g * nc;
    mr.wq_t = reinterpret_cast<i64 *>(mb);
    mr.hp_t = mr.wq_t + n;
    mr.wq_id = reinterpret_cast<u32 *>(mr.hp_t + nc);
    mr.hp_c = mr.wq_id + n;
    mr.nxr = mr.hp_c + nc;
    mr.ctok = mr.nxr + nc;
    mr.lprev = mr.ctok + nc;
    mr.lnext = mr.lprev + nc;
    mr.nconv = nc;
    mr.ntot = P.mr_ntot[g];
    mr.next0 = 0;
    mr.hsize = 0;
    mr.lhead = mr.ltail = MR_NIL;
    mr.used = 0;
    mr.cap = P.cache_cap ? P.cache_cap : 4 * total;
    #pragma unroll 1
    for (u32 x = lane; x < nc; x += 32) mr.ctok[x] = 0;
    __syncwarp();
  }
  u64 req_iters = 0, npre = 0, swo_tot = 0, swi_tot = 0, nrej_tot = 0, nfin_tot = 0, peak = 0, bns = 0;
  u64 ff_iters = 0, ff_runs = 0;
  u64 cyc_ff = 0, cyc_ff_fail = 0, cyc_normal = 0;
  long long clk_a = 0, clk_p = 0;
  u64 ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  u64 nph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  u32 ffr[5] = {0, 0, 0, 0, 0};  // failed fast-forward attempts: not quiet / memory / arrival / head / other
  u32 ffc[5] = {0, 0, 0, 0, 0};  // stretches ended by memory / a finish / an arrival / the head / 32 or other
#if TS_PROFILE
#define NPH(i)                           \
  do {                                   \
    const long long _c = clock64();      \
    nph[i] += (u64)(_c - clk_p);         \
    clk_p = _c;                          \
  } while (0)
#define PH(i)                            \
  do {                                   \
    const long long _c = clock64();      \
    ph[i] += (u64)(_c - clk_p);          \
    clk_p = _c;                          \
  } while (0)
#else
#define NPH(i) do {} while (0)
#define PH(i) do {} while (0)
#endif
  i64 last_fin = 0;
  u32 hd_idx = 0xffffffffu, hd_p = 0;  // cached prompt length of the fresh-queue head
  // memory trace state (lane-uniform)
  const bool BINNED = P.trace_mode == TOKENSIM_TRACE_BINNED;
  const bool FULLT = P.trace_mode == TOKENSIM_TRACE_FULL;
  const i64 W = (i64)P.bin_ns;
  u64 tn = 0, bin = 0, acc_bns = 0;
  i64 bin_end = W;
  u32 acc_max = 0, acc_nit = 0;
  FullEnc fe = {0, 0, 0, 0, 0, 0};  // FULL: the compressed stream (trace_codec.cuh)
  unsigned char *const tbuf = reinterpret_cast<unsigned char *>(trc);
  const u64 tcap_b = P.trace_cap * sizeof(tokensim_mem_sample);
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

  // request window: lane l holds arrival/prompt/output of request win + l
  u32 win = 0;
  i64 wa = INT64_MAX;
  u32 wp = 0, wo = 0;
  auto load_win = [&](u32 base) {
    win = base;
    const u32 i = base + lane;
    wa = i < n ? A[i] : INT64_MAX;
    wp = i < n ? PR[i] : 0u;
    wo = i < n ? OU[i] : 0u;
  };
  load_win(0);

  while (true) {
    // 0. termination
    if (MRM ? (mr.next0 == mr.nconv && mr.hsize == 0 && adm == arr && nR == 0 && nQ == 0)
            : (adm == n && nR == 0 && nQ == 0))
      break;
    if (P.horizon >= 0 && t >= P.horizon) {
      flags |= TOKENSIM_PT_HORIZON_HIT;
      break;
    }
    // 1. ingest: a_i <= t become visible at this boundary
    if (MRM) {
      // multi-round: the round-0 stream and pending follow-ups join the arrival FIFO in
      // (time, conversation) order; [adm, arr) of the FIFO is the fresh queue
      i64 ta;
      u32 cv;
      bool from0;
      while (mr_next(mr, A, ta, cv, from0) && ta <= t) {
        const u32 r = from0 ? 0u : mr.nxr[cv];
        if (from0) ++mr.next0;
        else mr_heap_pop(mr);
        mr.wq_id[arr] = mr.BASE[cv] + r;
        mr.wq_t[arr] = ta;
        ++arr;
      }
    } else {
      while (arr < n) {
        if (arr >= win + 32) load_win(arr);
        const u32 m = __ballot_sync(FULLMASK, (win + lane >= arr) && (wa <= t));
        arr += __popc(m);
        if (arr < win + 32) break;
      }
    }
    // 2. idle skip
    if (nR == 0 && nQ == 0 && adm == arr) {
      if (MRM) {
        i64 ta;
        u32 cv;
        bool from0;
        if (!mr_next(mr, A, ta, cv, from0)) {
          flags |= TOKENSIM_PT_INTERNAL_ERROR;
          break;
        }
        t = ta;
      } else {
        t = __shfl_sync(FULLMASK, wa, arr - win);
      }
      continue;
    }

    // ---------------------------------------------------------------- fast-forward (H3)
    clk_a = prof_clock();
    clk_p = clk_a;
    if (ff_on && nR > 0 && rmin >= 2 && !hx && (nfree > ff_mem_wait || k >= ff_mem_k)) {
      // The stretch must admit nothing and resume nothing.  With Q != {} fresh admission is
      // off (c.4 step 5) and a Q head that cannot resume now cannot resume later (R frozen,
      // free count only falls).  With Q = {}: STATIC never admits while R != {}; an empty fresh
      // queue is cut at the next arrival; a blocked fresh head stays blocked (step 5 is
      // monotone in the free count and the allocated count).
      bool quiet = true, mem_check = false;
      u32 need_h = 0;
      bool ratio_h = false;
      if (nQ > 0) {
        const u32 x = nR;  // Q head position
        u32 tokq;
        const u32 cq = S.ctx[x];
        if (SWAPM && !(CHK && cq == 0)) {
          need_h = B.cdiv(cq) + (B.mod(cq) == 0 ? 1u : 0u);
          tokq = 1;
        } else {
          const u32 id = S.id[x];
          tokq = PR[id] + (OU[id] - S.rem[x]);
          need_h = B.cdiv(tokq);
        }
        if (CHK) tokq = 1;  // one token of budget admits a chunk
        if (!((u64)nR + 1 > mns || (u64)nR + tokq > mbt)) {
          mem_check = true;
          // resume is certain even if every running request takes a block now: don't try
          if ((i64)nfree - (i64)nR - (i64)need_h >= wm) quiet = false;
        }
      } else if (!STATICP && adm < arr) {
        if (hd_idx != adm) {
          hd_idx = adm;
          const u32 off = adm - win;
          const u32 pw = __shfl_sync(FULLMASK, wp, off & 31u);
          hd_p = MRM ? PR[mr.wq_id[adm]] : ((adm >= win && off < 32) ? pw : PR[adm]);
        }
        need_h = B.cdiv(hd_p);
        // prefill-first admits before any decode block: no decode tokens, no decode blocks
        const u64 dtok = PFM ? 0u : nR;
        if ((u64)need_h > HP.cap_fresh) quiet = false;  // would be rejected at this boundary
        else if (!((u64)nR + 1 > mns || dtok + (CHK ? 1u : hd_p) > mbt)) {
          mem_check = true;
          ratio_h = RATIO;
          // admission is certain even if every running request takes a block now: don't try
          if ((i64)nfree - (i64)dtok - (i64)need_h >= wm &&
              (!RATIO || (total - nfree + dtok) + need_h <= HP.ratio_limit))
            quiet = false;
        }
      }
      // cheap predictors of a failed attempt (they only choose the path, never the result): the
      // running set needs about ceil(nR / bs) blocks per iteration -- with fewer free blocks the
      // stretch is cut at once by memory, and a head that still fits after that many is likely
      // admitted by the exact check below
      if (quiet) {
        const u64 est = B.cdiv(nR);
        if (nfree < est) quiet = false;
        else if (mem_check && (i64)nfree - (i64)est - (i64)need_h >= wm &&
                 (!ratio_h || (total - nfree + est) + need_h <= HP.ratio_limit))
          quiet = false;
      }
      if (quiet) {
        // C_d(0), min rem, and the needs histogram by iteration offset (lane j <-> iteration
        // k+j).  A slot needs a block at offsets j = j0 (mod bs), j0 = -ctx mod bs, so
        // n_j = cnt[j mod bs].  Right after another stretch all three are carried over (inc_*);
        // otherwise one pass over R counts slots per j0 with match_any (no atomics).
        u64 Cd0;
        u32 rm, hcl;
        if (XS && inc_ok) {
          Cd0 = inc_cd;
          rm = rmin;
          hcl = inc_h;
        } else {
          u64 cdp = 0;
          u32 rmn = 0xffffffffu;
          S.scratch[lane] = 0;
          S.scratch[32 + lane] = 0;
          __syncwarp();
          #pragma unroll 1
          for (u32 b0 = 0; b0 < nR; b0 += 32) {
            const u32 jj = b0 + lane;
            u32 key = 64u + lane;
            if (jj < nR) {
              const u32 c = S.ctx[jj];
              cdp += c + 1;
              rmn = min(rmn, S.rem[jj]);
              const u32 r = B.mod(c);
              const u32 j0 = r ? B.bs - r : 0u;
              if (j0 < 32) key = j0;
            }
            const u32 peers = __match_any_sync(FULLMASK, key);
            u32 old = 0;
            if (key < 32 && (peers & ltm) == 0u) {
              old = S.scratch[key];
              S.scratch[key] = old + __popc(peers);
              S.scratch[32 + key] = peers;  // slot positions of this residue (meaningful if nR <= 32)
            }
            // rank of the slot among the slots of its residue class, in position order (= its
            // place among the requesters of every iteration in which that class needs blocks)
            const u32 rbase = __shfl_sync(FULLMASK, old, (u32)(__ffs(peers) - 1));
            if (key < 32) S.req_pt[jj] = rbase + __popc(peers & ltm);
            __syncwarp();
          }
          Cd0 = warp_sum64(cdp);
          rm = __reduce_min_sync(FULLMASK, rmn);
          hcl = XS ? S.scratch[lane] : S.scratch[B.bs >= 32 ? lane : B.mod(lane)];
        }
        const u32 nj = XS ? __shfl_sync(FULLMASK, hcl, B.bs >= 32 ? lane : B.mod(lane)) : hcl;
        const u32 Aj = scan_incl(nj);  // cumulative blocks allocated through iteration k+lane
        PH(0);
        // lane-parallel cost of iteration k+lane: D = nR decodes, C_d grows by nR per iteration
        const u64 Cdj = Cd0 + (u64)lane * nR;
        const i64 Tj = iter_time_ns(K, 0, 0, 0, nR, Cdj, 0);
        // extended-stretch kernel: the second half's times in the same basic block (the two
        // evaluations and their scans interleave; unused when the first half is cut)
        i64 Tj1s = 0, sc1s = 0;
        if constexpr (XS && TS_SPEC) {
          Tj1s = iter_time_ns(K, 0, 0, 0, nR, Cd0 + (u64)(32u + lane) * nR, 0);
          sc1s = scan_incl_i64(Tj1s);
        }
        const i64 tej = t + scan_incl_i64(Tj);
        const i64 tsj = tej - Tj;
        // cut: the stretch is the longest prefix of iterations that stay quiescent; the
        // last one may finish requests (rem reaching 0), no earlier one may
        // (warp collectives stay outside lane-dependent branches)
        i64 a_next = __shfl_sync(FULLMASK, wa, (arr - win) & 31u);
        bool more = arr < n;
        if (MRM) {  // the next round-0 arrival or pending follow-up round
          u32 cv;
          bool f0;
          more = mr_next(mr, A, a_next, cv, f0);
        }
        bool ok = ((u64)Aj <= nfree) && (Aj <= (u32)CAP) && (lane < rm);
        u32 why = ((u64)Aj > nfree ? 1u : 0u) | (lane >= rm ? 2u : 0u);  // observability: cut reasons
        if (lane > 0) {
          if (P.horizon >= 0 && tsj >= P.horizon) ok = false;
          if (nQ == 0 && adm == arr && more && tsj >= a_next) {
            ok = false;
            why |= 4u;
          }
        }
        if (mem_check) {  // head blocked by memory at this boundary? (then for the whole stretch)
          const u64 n0 = (u64)__shfl_sync(FULLMASK, Aj, 0);
          const u64 fr = nfree - ((PFM && nQ == 0) ? 0ull : n0);
          const bool blocked = ((i64)fr - (i64)need_h < wm) || (ratio_h && (total - fr) + need_h > HP.ratio_limit);
          if (!blocked) {
            ok = false;
            why |= 8u;
          }
        }
        const u32 okm = __ballot_sync(FULLMASK, ok);
        u32 J = (~okm == 0u) ? 32u : (u32)(__ffs(~okm) - 1);
        // Second half (iterations k+32+lane, block sizes <= 32 only so the needs histogram
        // covers them): evaluated only when all 32 of the first half pass, so a stretch of up to
        // 64 iterations costs one pass over R, one set of slot updates and one log publication
        // instead of two.  Values of iteration j >= 32 are the *1 registers on lane j - 32.
        u32 nj1 = 0, Aj1 = 0;
        u64 Cdj1 = 0;
        i64 Tj1 = 0, tej1 = 0, tsj1 = 0;
        if (XS && J == 32 && B.bs <= 32u) {
          nj1 = __shfl_sync(FULLMASK, hcl, B.mod(32u + lane) & 31u);
          Aj1 = __shfl_sync(FULLMASK, Aj, 31) + scan_incl(nj1);
          Cdj1 = Cd0 + (u64)(32u + lane) * nR;
          if constexpr (TS_SPEC) {
            Tj1 = Tj1s;
            tej1 = __shfl_sync(FULLMASK, tej, 31) + sc1s;
          } else {
            Tj1 = iter_time_ns(K, 0, 0, 0, nR, Cdj1, 0);
            tej1 = __shfl_sync(FULLMASK, tej, 31) + scan_incl_i64(Tj1);
          }
          tsj1 = tej1 - Tj1;
          bool ok1 = ((u64)Aj1 <= nfree) && (Aj1 <= (u32)CAP) && (32u + lane < rm);
          if (P.horizon >= 0 && tsj1 >= P.horizon) ok1 = false;
          if (nQ == 0 && adm == arr && more && tsj1 >= a_next) ok1 = false;
          const u32 okm1 = __ballot_sync(FULLMASK, ok1);
          J = 32u + ((~okm1 == 0u) ? 32u : (u32)(__ffs(~okm1) - 1));
        }
        const bool two = XS && J > 32u;
        if (!TS_PROFILE) {
        } else if (J < 2) {
          const u32 w = __shfl_sync(FULLMASK, why, J);
          ffr[(w & 1u) ? 1 : (w & 4u) ? 2 : (w & 8u) ? 3 : 4] += 1;
        } else {  // what ended a stretch: memory / a finish / an arrival / the head / 32 or other
          const u32 w = J < 32 ? __shfl_sync(FULLMASK, why, J) : 0u;  // (second-half cuts: "other")
          ffc[(w & 1u) ? 0 : (w & 2u) ? 1 : (w & 4u) ? 2 : (w & 8u) ? 3 : 4] += 1;
        }
        // a stretch cut short by memory will not grow until blocks come back: remember the level
        const u32 memcut = __ballot_sync(FULLMASK, !((u64)Aj <= nfree));
        if (J < 2 && memcut && (u32)(__ffs(memcut) - 1) < 2) {
          ff_mem_wait = nfree;
          ff_mem_k = k + 4;  // the needs pattern shifts with the ctx residues: retry soon anyway
        }
        if (J >= 2) {
          const u32 Ktot = __shfl_sync(FULLMASK, two ? Aj1 : Aj, (J - 1) & 31u);
          PH(1);
          bool done_alloc = Ktot == 0;
          if (!HEV && !TS_NO_FUSED && !done_alloc && !two && nR <= 32 && Ktot <= 32 && hint < nwords) {
            // fused small case: lane o takes the o-th lowest free block of the 32-word window at
            // the hint and serves order index o = (iteration jb, r-th slot of jb's residue class)
            const u32 wi = hint + lane;
            u32 word = wi < nwords ? S.bitmap[wi] : 0u;
            const u32 cw = __popc(word);
            const u32 cum = scan_incl(cw);
            if (__shfl_sync(FULLMASK, cum, 31) >= Ktot) {
              ev_reserve(L, 32);
              const bool act = lane < Ktot;
              const u32 o = act ? lane : 0u;
              u32 jb = 0;
#pragma unroll
              for (u32 st = 16; st; st >>= 1) {
                const u32 v = __shfl_sync(FULLMASK, Aj, jb + st - 1);
                if (v <= o) jb += st;
              }
              const u32 excl = __shfl_sync(FULLMASK, Aj - nj, jb);
              u32 lo = 0;
#pragma unroll
              for (u32 st = 16; st; st >>= 1) {
                const u32 v = __shfl_sync(FULLMASK, cum, lo + st - 1);
                if (v <= o) lo += st;
              }
              const u32 wv = __shfl_sync(FULLMASK, word, lo);
              const u32 bv = __shfl_sync(FULLMASK, cum - cw, lo);
              if (act) {
                const u32 mask = S.scratch[32 + (B.bs >= 32 ? jb : B.mod(jb))];
                const u32 pos = select_bit(mask, o - excl);
                const u32 blk = (hint + lo) * 32 + select_bit(wv, o - bv);
                const u32 tpos = B.div(S.ctx[pos] + jb);
                bt[(size_t)(SLOT(S.info[pos])) * btl + tpos] = blk;
                ev_put(L, o, k + jb, 1, S.id[pos], blk);
              }
              L.nev += Ktot;
              const u32 before = cum - cw;
              const u32 tk = Ktot > before ? min(cw, Ktot - before) : 0u;
              if (tk && wi < nwords) {
                word = clear_lowest(word, tk, cw);
                S.bitmap[wi] = word;
              }
              const u32 nz = __ballot_sync(FULLMASK, word != 0u);
              hint = nz ? hint + (u32)(__ffs(nz) - 1) : hint + 32;
              __syncwarp();
              done_alloc = true;
            }
          }
          if (!done_alloc) {
            // the Ktot lowest free blocks in order, then every request places itself: the
            // request of a slot at iteration offset jx has order index (blocks of iterations
            // before jx) + (its rank in its residue class)
            u32 *fl = S.req_cum;  // free in a stretch; Ktot <= CAP (cut condition)
            if (HEV) {
              ev_begin(Ktot);
            } else {
              if (!take_lowest(S.bitmap, Ktot, fl, hint, nwords)) {
                flags |= TOKENSIM_PT_INTERNAL_ERROR;
                break;
              }
              ev_reserve(L, Ktot);
            }
            const u32 excl = Aj - nj, excl1 = Aj1 - nj1;
            const u32 nrep = B.cdiv(XS ? J : 32u);  // (shifts when bs is a power of two)
            #pragma unroll 1
            for (u32 b0 = 0; b0 < nR; b0 += 32) {
              const u32 jj = b0 + lane;
              const bool in = jj < nR;
              const u32 c = in ? S.ctx[jj] : 0u;
              const u32 rank = in ? S.req_pt[jj] : 0u;
              const u32 r = B.mod(c);
              u32 jx = r ? B.bs - r : 0u;
              #pragma unroll 1
              for (u32 rep = 0; rep < nrep; ++rep, jx += B.bs) {
                const u32 ex0 = __shfl_sync(FULLMASK, excl, jx & 31u);
                const u32 ex1 = two ? __shfl_sync(FULLMASK, excl1, jx & 31u) : 0u;  // (uniform branch)
                const u32 ex = jx < 32u ? ex0 : ex1;
                if (in && jx < J) {
                  const u32 o = ex + rank;
                  if (HEV) {
                    ev_log(o, k + jx, HEV_ALLOC, 1, S.id[jj], SLOT(S.info[jj]), B.div(c + jx));
                  } else {
                    const u32 blk = fl[o];
                    bt[(size_t)SLOT(S.info[jj]) * btl + B.div(c + jx)] = blk;
                    ev_put(L, o, k + jx, 1, S.id[jj], blk);
                  }
                }
              }
            }
            L.nev += Ktot;
            __syncwarp();
          }
          const u64 blk0 = total - nfree;
          nfree -= Ktot;
          const u64 klast = k + J - 1;
          PH(2);
          // slot updates for J decode iterations; requests reaching rem == 0 finish in the last
          const i64 tend = __shfl_sync(FULLMASK, two ? tej1 : tej, (J - 1) & 31u);
          const i64 tsl = __shfl_sync(FULLMASK, two ? tsj1 : tsj, (J - 1) & 31u);
          const bool lj = lane < J;               // first-half iterations of the stretch
          const bool lj1 = two && 32u + lane < J;  // second-half iterations
          // the largest gap of the stretch is its last iteration's: T_j is nondecreasing in j
          // (only C_d grows, and every rounded product, sum, fmax and floor in the cost model is
          // monotone in it with nonnegative coefficients), so max_{j<J} T_j = T_{J-1}
          const i64 tmax = tend - tsl;
          u32 nfin = 0, first_fin = 0xffffffffu, rmin_l = 0xffffffffu;
          // carried state: every slot advanced J tokens (the histogram rotates by J); finished
          // slots leave R below
          u64 cd_next = Cd0 + (u64)J * nR;
          u32 h_next = 0;
          if constexpr (XS) h_next = __shfl_sync(FULLMASK, hcl, B.mod(lane + J) & 31u);  // bs <= 32 (else unused)
          #pragma unroll 1
          for (u32 b0 = 0; b0 < nR; b0 += 32) {
            const u32 jj = b0 + lane;
            bool fin = false;
            if (jj < nR) {
              const u32 r = S.rem[jj] - J;
              S.rem[jj] = r;
              S.ctx[jj] += J;
              const i64 mg = tmax > S.maxgap[jj] ? tmax : S.maxgap[jj];
              S.maxgap[jj] = mg;
              S.last[jj] = tend;
              fin = r == 0;
              if (fin) {
                const u32 id = S.id[jj];
                const i64 ttft = S.ttft[jj], e2e = tend - S.arr[jj];
                const u32 np_ = S.info[jj] >> 16;
                write_record(rec + id, ttft, e2e, mg, np_, TOKENSIM_REQ_FINISHED, (u32)klast);
              } else {
                rmin_l = min(rmin_l, r);
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
              const u32 cf = S.ctx[pos];
              const u32 held = B.cdiv(cf);
              const u32 slot = SLOT(S.info[pos]);
              if constexpr (XS) {
                cd_next -= cf + 1;
                const u32 rf = B.mod(cf);
                if (lane == (rf ? B.bs - rf : 0u)) h_next -= 1;
              }
              if (HEV) ev_free(held, S.id[pos], slot, klast);
              else free_blocks(S.bitmap, bt + (size_t)slot * btl, held, S.id[pos], klast, 0, L, hint);
              nfree += held;
              if (lane == 0) atomicOr(&S.btfree[slot >> 5], 1u << (slot & 31u));
              if (MRM) {  // NEXT-2: store the context; schedule the conversation's next round
                const u32 rid = S.id[pos];
                const u32 cv = mr.CONV[rid];
                const u32 r = rid - mr.BASE[cv];
                if (CACHE) mr_cache_store(mr, cv, PR[rid] + OU[rid] - 1u, B);
                if (r + 1 < mr.NR[cv]) {
                  mr.nxr[cv] = r + 1;
                  mr_heap_push(mr, tend + A[rid + 1], cv);
                }
                __syncwarp();
              }
            }
          }
          __syncwarp();
          PH(3);
          // iteration records, digests, counters (lanes j < J)
          const u64 blkj = blk0 + Aj, blkj1 = blk0 + Aj1;
          it_begin(XS ? 64u : 32u);
          if (lj) it_put(L, lane, k + lane, tsj, Tj, 0, Cdj, blkj, 0, nR, 0, 0, 0, lane == J - 1 ? nfin : 0u, 0);
          if (lj1)
            it_put(L, 32u + lane, k + 32u + lane, tsj1, Tj1, 0, Cdj1, blkj1, 0, nR, 0, 0, 0,
                   32u + lane == J - 1 ? nfin : 0u, 0);
          L.nit += J;
          it_commit();
          const u64 bns_add =
              HELP ? 0ull : warp_sum64((lj ? blkj * (u64)Tj : 0ull) + (lj1 ? blkj1 * (u64)Tj1 : 0ull));
          PH(4);
          // memory trace
          if (HELP) {
          } else if (BINNED) {
            while (true) {
              const i64 bstart = bin_end - W;
              i64 ov = 0, ov1 = 0;
              bool cnt_here = false, cnt1 = false;
              if (lj) {
                const i64 lo = tsj > bstart ? tsj : bstart;
                const i64 hi = tej < bin_end ? tej : bin_end;
                ov = hi - lo;
                cnt_here = tsj >= bstart && tsj < bin_end;
              }
              if (lj1) {
                const i64 lo = tsj1 > bstart ? tsj1 : bstart;
                const i64 hi = tej1 < bin_end ? tej1 : bin_end;
                ov1 = hi - lo;
                cnt1 = tsj1 >= bstart && tsj1 < bin_end;
              }
              const u64 add = warp_sum64((ov > 0 ? blkj * (u64)ov : 0ull) + (ov1 > 0 ? blkj1 * (u64)ov1 : 0ull));
              const u32 mx = __reduce_max_sync(FULLMASK, max(ov > 0 ? (u32)blkj : 0u, ov1 > 0 ? (u32)blkj1 : 0u));
              acc_bns += add;
              acc_max = max(acc_max, mx);
              acc_nit += __popc(__ballot_sync(FULLMASK, cnt_here)) + __popc(__ballot_sync(FULLMASK, cnt1));
              if (tend > bin_end || tsl >= bin_end) flush_bin();
              else break;
            }
          } else if (FULLT) {
            full_trace_put(fe, tbuf, tcap_b, two ? 32u : J, tsj, tsj + Tj, blkj, flags);
            if (two) full_trace_put(fe, tbuf, tcap_b, J - 32u, tsj1, tsj1 + Tj1, blkj1, flags);
          }
          if (!HELP) {
            const u64 blk_last = blk0 + Ktot;
            peak = blk_last > peak ? blk_last : peak;
            bns += bns_add;
          }
          req_iters += (u64)nR * J;
          PH(5);
          if (nfin) {
            const u32 len = nR + nQ;
            u32 out = first_fin;
            #pragma unroll 1
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
            last_fin = tend;
          }
          PH(6);
          rmin = nR ? __reduce_min_sync(FULLMASK, rmin_l) : 0u;
          // ranks within a residue class (S.req_pt) survive the rotation while no slot left R;
          // a finish compacts the slots, and the next stretch recounts
          inc_ok = XS && B.bs <= 32u && nfin == 0;
          inc_cd = cd_next;
          inc_h = h_next;
          PH(7);
          ff_iters += J;
          ++ff_runs;
          t = tend;
          k += J;
          cyc_ff += (u64)(prof_clock() - clk_a);
          continue;
        }
      }
      if (TS_PROFILE && !quiet) ffr[0] += 1;
      rmin = 0;  // retry only after the next normal commit recomputes it
      const long long c1 = prof_clock();
      cyc_ff_fail += (u64)(c1 - clk_a);
      clk_a = c1;
    }
    clk_p = prof_clock();
    inc_ok = false;  // a normal iteration changes R and the contexts: the next stretch recounts

    // ---------------------------------------------------------------- 3. decode reservation
    u32 E = 0, Kb = 0, m = 0, nres = 0, nadm = 0, nrej = 0, Edec = 0;
    u64 cdp = 0, npp = 0, app = 0, swap_out = 0, swap_in = 0, tokens = 0;
    // CHUNKED: keys read by prefills, LM-head rows, the entry left partial this iteration
    u64 kpp = 0;
    u32 semit = 0, nres_sw = 0;
    u64 fetch_blocks = 0;  // NEXT-2: cached blocks fetched by this iteration's hits
    bool hnew = false;
    u32 xnew_pos = 0, xnew_done = 0, xnew_tgt = 0;
    auto note_partial = [&](bool part, u32 pos, u32 ch, u32 tgt) {
      const u32 pm = __ballot_sync(FULLMASK, part);
      if (pm) {
        const int src = __ffs(pm) - 1;
        hnew = true;
        xnew_pos = __shfl_sync(FULLMASK, pos, src);
        xnew_done = __shfl_sync(FULLMASK, ch, src);
        xnew_tgt = __shfl_sync(FULLMASK, tgt, src);
      }
    };
    // 5. fresh FCFS admission (its own pass in prefill-first mode, NEXT-3)
    auto fresh_admit = [&]() {
      bool head_blocked = false;
      if (adm < arr) {
        // quick exit: a head that is not rejected but cannot be admitted stops step 5 at once
        const u32 off = adm - win;
        const u32 pw = __shfl_sync(FULLMASK, wp, off & 31u);
        const u32 ph = MRM ? PR[mr.wq_id[adm]] : ((adm >= win && off < 32) ? pw : PR[adm]);
        const u32 nh = B.cdiv(ph);
        head_blocked = !TS_AB_NO_HEADQ && (u64)nh <= HP.cap_fresh &&
                       ((u64)nR + 1 > mns || tokens + (CHK ? 1u : ph) > (u64)mbt || (i64)nfree - (i64)nh < wm ||
                        (RATIO && (total - nfree) + nh > HP.ratio_limit));
      }
      if (!head_blocked) {
        while (adm < arr) {
          const u32 i = adm + lane;
          const bool valid = i < arr;
          const u32 off = i - win;
          const bool inw = i >= win && off < 32;
          u32 p = __shfl_sync(FULLMASK, wp, off & 31u);
          u32 o = __shfl_sync(FULLMASK, wo, off & 31u);
          i64 a = __shfl_sync(FULLMASK, wa, off & 31u);
          u32 rid = i;  // request id (multi-round: from the arrival FIFO)
          if (!valid) {
            p = 0;
            o = 0;
            a = 0;
          } else if (MRM) {
            rid = mr.wq_id[i];
            p = PR[rid];
            o = OU[rid];
            a = mr.wq_t[i];
          } else if (!inw) {
            p = PR[i];
            o = OU[i];
            a = A[i];
          }
          const u32 need = B.cdiv(p);
          const bool rej = valid && (u64)need > HP.cap_fresh;
          const bool el = valid && !rej;
          // one candidate (the common case at low load): lane 0's prefix sums are its own values,
          // and every other lane's are masked by !el below, so the three scans are skipped
          const bool one = !TS_AB_NO_ONEADM && arr - adm == 1u;
          const u32 ce = one ? (el ? 1u : 0u) : scan_incl(el ? 1u : 0u);
          const u32 cneed = one ? (el ? need : 0u) : scan_incl(el ? need : 0u);
          const u32 cp = one ? (el ? p : 0u) : scan_incl(el ? p : 0u);
          // CHUNKED: a request is admitted while one token of budget is left (reading R-N3b)
          const bool tok_ok = CHK ? tokens + cp - p < (u64)mbt : tokens + cp <= (u64)mbt;
          const bool ok = el && ((u64)nR + ce <= (u64)mns) && tok_ok &&
                          ((i64)nfree - (i64)cneed >= wm) && (!RATIO || (total - nfree) + cneed <= HP.ratio_limit);
          const u32 failm = __ballot_sync(FULLMASK, el && !ok);
          const u32 nvalid = min(32u, arr - adm);
          const u32 stop = failm ? (u32)(__ffs(failm) - 1) : nvalid;
          const bool take = el && lane < stop;
          const bool rj = rej && lane < stop;
          const u32 takem = __ballot_sync(FULLMASK, take);
          const u32 cnt = __popc(takem);
          // NEXT-2 cache lookups, in admission order: a later round of a cached conversation
          // skips its cached prefix c0 and pays the fetch of its blocks (reading R-N2)
          u32 c0 = 0;
          if (CACHE && cnt) {
            u32 tm = takem;
            while (tm) {
              const u32 l = (u32)(__ffs(tm) - 1);
              tm &= tm - 1;
              const u32 lrid = __shfl_sync(FULLMASK, rid, l);
              const u32 cv = mr.CONV[lrid];
              u32 hit = 0;
              if (lrid > mr.BASE[cv] && mr.ctok[cv]) {
                hit = mr.ctok[cv];
                fetch_blocks += B.cdiv(hit);
                mr_unlink(mr, cv);
                mr_append(mr, cv);
              }
              if (lane == l) c0 = hit;
            }
            __syncwarp();
          }
          if (cnt) {
            const u32 rank = __popc(takem & ltm);
            const u32 slot = alloc_btslots(S.btfree, CAP / 32, take, rank, cnt);
            u32 ch = p - c0;
            if (CHK && take) ch = (u32)min((u64)p, (u64)mbt - (tokens + cp - p));
            if (take) {
              const u32 pos = nR + rank;
              S.id[pos] = rid;
              S.ctx[pos] = p;  // fresh prefill of P = p; ctx after commit
              S.rem[pos] = o;
              S.info[pos] = CHK ? (slot | INFO_NT) : slot;
              S.last[pos] = 0;
              S.maxgap[pos] = 0;
              S.arr[pos] = a;
              S.ttft[pos] = 0;
              S.req_cum[E + rank] = Kb + cneed;
              S.req_pt[E + rank] = pos;
              npp += ch;
              app += (u64)ch * c0 + (u64)ch * (ch + 1) / 2;
              kpp += (u64)c0 + ch;
              semit += ch == p ? 1u : 0u;
            }
            if (CHK) note_partial(take && ch < p, nR + rank, ch, p);
          }
          if (rj) reinterpret_cast<uint8_t *>(rec + rid)[26] = (uint8_t)TOKENSIM_REQ_REJECTED;
          u32 nrj = __popc(__ballot_sync(FULLMASK, rj));
          if (MRM) {  // a rejected round ends its conversation: its later rounds never arrive
            u32 rm = __ballot_sync(FULLMASK, rj);
            while (rm) {
              const u32 l = (u32)(__ffs(rm) - 1);
              rm &= rm - 1;
              const u32 lrid = __shfl_sync(FULLMASK, rid, l);
              const u32 cv = mr.CONV[lrid];
              const u32 last = mr.BASE[cv] + mr.NR[cv];
              #pragma unroll 1
              for (u32 q = lrid + 1 + lane; q < last; q += 32)
                reinterpret_cast<uint8_t *>(rec + q)[26] = (uint8_t)TOKENSIM_REQ_REJECTED;
              nrj += last - lrid - 1;
            }
          }
          if (stop) {
            const u32 sneed = __shfl_sync(FULLMASK, cneed, stop - 1);
            const u32 sp = __shfl_sync(FULLMASK, cp, stop - 1);
            nfree -= sneed;
            Kb += sneed;
            tokens = CHK ? min(tokens + sp, (u64)mbt) : tokens + sp;
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
    };
    const u32 nR_old = nR;
    bool pf_only = false;
    if (PFM && nQ == 0 && (!STATICP || nR == 0)) {  // prefill-first: fresh prefills alone, if any
      fresh_admit();
      pf_only = nadm > 0;
    }
    u32 nR3 = nR_old;  // fresh prefills of a prefill-first iteration start at nR_old
    u32 chx = 0;        // CHUNKED: chunk of the prefill in progress (0: it sits this one out)
    bool xpart = false;  // ... and it stays partial
    if (!pf_only) {
    // one pass: needing survivors -> requester list (ascending id), sum of c = ctx+1
    #pragma unroll 1
    for (u32 b0 = 0; b0 < nR; b0 += 32) {
      const u32 jj = b0 + lane;
      const bool dec = jj < nR && !(hx && jj == nR - 1);  // the prefill in progress decodes nothing
      const u32 c = dec ? S.ctx[jj] : 1u;
      const bool need = dec && B.mod(c) == 0;
      if (dec) cdp += c + 1;
      const u32 bal = __ballot_sync(FULLMASK, need);
      if (need) {
        const u32 e = E + __popc(bal & ltm);
        S.req_cum[e] = e + 1;
        S.req_pt[e] = jj | (B.div(c) << 15);
      }
      E += __popc(bal);
    }
    if ((u64)E > nfree) {
      // minimal m with sum_{j<=n-m} need_j <= F + sum_{j>n-m} held_j (SURVEY c.4 step 3)
      u64 Sn = E, Hh = 0;
      do {
        ++m;
        const u32 c = S.ctx[nR - m];  // ctx = target of a prefill in progress: its held blocks
        Sn -= (B.mod(c) == 0 && !(hx && m == 1)) ? 1 : 0;
        Hh += B.cdiv(c);
      } while (Sn > nfree + Hh);
      u64 csub = 0;
      for (u32 v = nR - m; v < nR; ++v) {  // victims: latest arrivals (reading A7)
        const u32 c = S.ctx[v];
        const u32 held = B.cdiv(c);
        const u32 slot = SLOT(S.info[v]);
        // a partial prefill loses its KV whatever the mode: re-prefill from scratch (R-N3b)
        const bool vx = hx && v == nR - 1;
        if (HEV) ev_free(held, S.id[v], slot, k);
        else free_blocks(S.bitmap, bt + (size_t)slot * btl, held, S.id[v], k, 0, L, hint);
        nfree += held;
        if (!vx) csub += c + 1;
        if (SWAPM && !vx) swap_out += (u64)held * HP.block_bytes;
        __syncwarp();
        if (lane == 0) {
          S.info[v] += 1u << 16;
          if (!SWAPM || vx) S.ctx[v] = 0;
        }
      }
      hx = false;  // a prefill in progress is the tail of R: always the first victim
      __syncwarp();
      if (lane == 0) cdp -= csub;
      E = (u32)Sn;  // the requester list is in position order: victims are its tail
      nR -= m;
      nQ += m;
      npre += m;
    }
    nR3 = nR;
    Kb = E;
    Edec = E;  // decode requesters: one block each, first in phase order
    nfree -= E;
    tokens = nR - (hx ? 1u : 0u);
    if (CHK && hx) {  // the prefill in progress takes the budget the decodes leave (R-N3b)
      const u32 rest = xtgt - xdone;
      chx = (u32)min((u64)rest, (u64)mbt - tokens);
      xpart = chx < rest;
      if (lane == 0 && chx) {
        npp += chx;
        app += (u64)chx * xdone + (u64)chx * (chx + 1) / 2;
        kpp += (u64)xdone + chx;
        semit += xpart ? 0u : 1u;
      }
      tokens += chx;
    }
    if (m == 0) {
      NPH(0);
      // 4. resume, head first, stop at the first misfit
      if (nQ > 0) {
        u64 cum_need = 0, cum_tok = 0;
        #pragma unroll 1
        for (u32 b0 = 0; b0 < nQ; b0 += 32) {
          const u32 jj = nR3 + b0 + lane;
          const bool valid = b0 + lane < nQ;
          u32 need = 0, tok = 0, held0 = 0, c = 0;
          bool isrc = false;  // re-prefill p + gen (RECOMPUTE; CHUNKED: a lost partial prefill)
          if (valid) {
            c = S.ctx[jj];
            if (SWAPM && !(CHK && c == 0)) {
              need = B.cdiv(c) + (B.mod(c) == 0 ? 1u : 0u);
              tok = 1;
              held0 = B.cdiv(c);
            } else {
              const u32 id = S.id[jj];
              const u32 Pq = PR[id] + (OU[id] - S.rem[jj]);  // p + gen
              need = B.cdiv(Pq);
              tok = Pq;
              isrc = true;
            }
          }
          const u32 cn = scan_incl(need), ct = scan_incl(tok);
          const bool tok_ok = CHK ? tokens + cum_tok + ct - tok < (u64)mbt : tokens + cum_tok + ct <= (u64)mbt;
          const bool ok = valid && ((u64)nR3 + b0 + lane + 1 <= (u64)mns) && tok_ok &&
                          ((i64)nfree - (i64)(cum_need + cn) >= wm);
          const u32 okm = __ballot_sync(FULLMASK, ok);
          const u32 cnt = (~okm == 0u) ? 32u : (u32)(__ffs(~okm) - 1);
          u32 ch = tok;
          if (lane < cnt) {
            S.req_cum[E + lane] = Kb + cn;
            S.req_pt[E + lane] = jj;
            if (!isrc) {
              cdp += c + 1;
            } else {
              if (CHK) {
                ch = (u32)min((u64)tok, (u64)mbt - (tokens + cum_tok + ct - tok));
                S.info[jj] |= INFO_PFB;
              }
              S.ctx[jj] = tok;  // recompute prefill of P = p + gen; ctx after commit
              npp += ch;
              app += (u64)ch * (ch + 1) / 2;
              kpp += ch;
              semit += ch == tok ? 1u : 0u;
            }
          }
          if (CHK) {
            note_partial(lane < cnt && isrc && ch < tok, jj, ch, tok);
            nres_sw += __popc(__ballot_sync(FULLMASK, lane < cnt && !isrc));
          } else if (SWAPM) {
            nres_sw += cnt;
          }
          const u64 sw = warp_sum64(lane < cnt ? (u64)held0 : 0ull);
          if (cnt) {
            const u32 sn = __shfl_sync(FULLMASK, cn, cnt - 1), stk = __shfl_sync(FULLMASK, ct, cnt - 1);
            cum_need += sn;
            cum_tok += stk;
            Kb += sn;
            E += cnt;
            nres += cnt;
            if (SWAPM) swap_in += sw * HP.block_bytes;
          }
          if (cnt < 32) break;
        }
        nfree -= cum_need;
        tokens = CHK ? min(tokens + cum_tok, (u64)mbt) : tokens + cum_tok;
        nR += nres;
        nQ -= nres;
        __syncwarp();
      }
      NPH(1);
      if (!PFM && nQ == 0 && (!STATICP || nR == 0)) fresh_admit();
    }
    }
    nrej_tot += nrej;
    NPH(2);
    // 6. empty batch (every candidate rejected): back to 0 without advancing t
    if (nR == 0) continue;
    // block extraction for all requesters of this iteration, in phase order
    if (HEV) {
      if (Kb > 0) {  // one event per requester entry, in phase order
        #pragma unroll 1
        for (u32 e0 = 0; e0 < E; e0 += 32) {
          const u32 cnt = min(32u, E - e0);
          ev_begin(cnt);
          const u32 e = e0 + lane;
          if (e < E) {
            const u32 pt = S.req_pt[e];
            const u32 pos = PT_POS(pt);
            const u32 c1 = S.req_cum[e] - (e ? S.req_cum[e - 1] : 0u);
            ev_log(lane, k + PT_J(pt), HEV_ALLOC, c1, S.id[pos], SLOT(S.info[pos]), PT_TPOS(pt));
          }
          L.nev += cnt;
        }
      }
    } else if (Kb > 0 && !alloc_ordered(S, E, Kb, bt, btl, k, 0, L, hint, nwords, Edec)) {
      flags |= TOKENSIM_PT_INTERNAL_ERROR;
      break;
    }
    NPH(3);
    // 7. cost: decodes are positions [0, D), prefills [D, nR); a prefill-first iteration runs
    // only the fresh prefills at [nR_old, nR)
    // CHUNKED: the prefill in progress (position nR3 - 1 when hx) is not a decode; with chx = 0
    // it is not in the batch at all
    const bool xout = hx && chx == 0;
    const u32 D = pf_only ? 0u : nR3 - (hx ? 1u : 0u) + nres_sw;
    const u32 Sp = pf_only ? nR - nR_old : nR - D - (xout ? 1u : 0u);
    const u32 c0 = pf_only ? nR_old : 0u;
    const u64 Cd = warp_sum64(cdp);
    u64 Np = 0, Ap = 0, Kp = 0, Slm = Sp;
    if (Sp) {
      // lean kernels (MIXED): every prefill token was admitted under tokens <= mbt (a u32), so
      // N_p < 2^32 and one 32-bit reduction is exact
      Np = FULL ? warp_sum64(npp) : (u64)__reduce_add_sync(FULLMASK, (u32)npp);
      Ap = warp_sum64(app);
      Kp = Np;
      if (CHK || CACHE) Kp = warp_sum64(kpp);
      if (CHK) Slm = __reduce_add_sync(FULLMASK, semit);
    }
    // the preload pipeline's scratch: the block-event log (flushed first), or -- when the helper
    // warp consumes that log -- a per-warp region of its own
    double *pring = HELP ? P.pipe + (size_t)gwarp * P.pipe_stride : reinterpret_cast<double *>(L.ev);
    if (!HELP && K.preload && swap_in > 0) ev_flush(L);
    const i64 T = iter_time_chunk_ns(K, Np, Ap, Kp, Slm, D, Cd, swap_out, swap_in, pring,
                                     fetch_blocks);
    NPH(4);
    // 8. commit
    const i64 ts = t, te = t + T;
    const u64 blocks = total - nfree;
    u32 nfin = 0, first_fin = 0xffffffffu, rmin_l = 0xffffffffu;
    const u32 fresh0 = nR3 + nres;
    // CHUNKED: position of the entry whose prefill stays partial (no token this iteration)
    const u32 ppos = (hx && xpart) ? nR3 - 1 : (hnew ? xnew_pos : 0xffffffffu);
    #pragma unroll 1
    for (u32 b0 = c0; b0 < nR; b0 += 32) {
      const u32 jj = b0 + lane;
      bool fin = false;
      if (CHK) {
        if (jj < nR) {
          const u32 inf = S.info[jj];
          const bool isx = hx && jj == nR3 - 1;
          const bool emit = jj != ppos && !(isx && chx == 0);
          const bool dec = (jj < nR3 && !isx) || (jj >= nR3 && jj < fresh0 && !(inf & INFO_PFB));
          u32 r = S.rem[jj];
          if (emit) {
            r -= 1;
            S.rem[jj] = r;
            if (dec) S.ctx[jj] += 1;
            if (inf & INFO_NT) {  // the first token
              S.ttft[jj] = te - S.arr[jj];
            } else {
              const i64 gap = te - S.last[jj];
              if (gap > S.maxgap[jj]) S.maxgap[jj] = gap;
            }
            S.last[jj] = te;
            if (inf & (INFO_NT | INFO_PFB)) S.info[jj] = inf & ~(INFO_NT | INFO_PFB);
          } else if (inf & INFO_PFB) {
            S.info[jj] = inf & ~INFO_PFB;
          }
          fin = emit && r == 0;
          if (fin) {
            write_record(rec + S.id[jj], S.ttft[jj], te - S.arr[jj], S.maxgap[jj], S.info[jj] >> 16,
                         TOKENSIM_REQ_FINISHED, (u32)k);
          } else {
            rmin_l = min(rmin_l, r);
          }
        }
      } else if (jj < nR) {
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
        } else {
          rmin_l = min(rmin_l, r);
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
        const u32 held = B.cdiv(c);
        const u32 slot = SLOT(S.info[pos]);
        if (HEV) ev_free(held, S.id[pos], slot, k);
        else free_blocks(S.bitmap, bt + (size_t)slot * btl, held, S.id[pos], k, 0, L, hint);
        nfree += held;
        if (lane == 0) atomicOr(&S.btfree[slot >> 5], 1u << (slot & 31u));
        if (MRM) {  // NEXT-2: store the context; schedule the conversation's next round
          const u32 rid = S.id[pos];
          const u32 cv = mr.CONV[rid];
          const u32 r = rid - mr.BASE[cv];
          if (CACHE) mr_cache_store(mr, cv, PR[rid] + OU[rid] - 1u, B);
          if (r + 1 < mr.NR[cv]) {
            mr.nxr[cv] = r + 1;
            mr_heap_push(mr, te + A[rid + 1], cv);
          }
          __syncwarp();
        }
      }
    }
    NPH(5);
    {
      const u32 rn = __reduce_min_sync(FULLMASK, rmin_l);
      // After a prefill-only iteration the paused decodes' last token is older than t, so the
      // next stretch's first gap would exceed its last iteration's T (the stretch takes T_{J-1}
      // as every slot's largest gap): no stretch until a normal iteration has given every
      // running request a token at t.
      rmin = pf_only ? 0u : rn;
    }
    __syncwarp();
    req_iters += nR - c0 - (xout ? 1u : 0u);
    if (CHK) {  // the prefill in progress after this iteration (R-N3b)
      if (hx && !xout) {
        if (xpart) xdone += chx;
        else hx = false;
      }
      if (hnew) {
        hx = true;
        xdone = xnew_done;
        xtgt = xnew_tgt;
      }
    }
    NPH(6);
    if (nfin) {
      // stable compaction of R u Q, dropping finished entries (rem == 0 within R)
      const u32 len = nR + nQ;
      u32 out = first_fin;
      #pragma unroll 1
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
    if (nR == 0) rmin = 0;
    NPH(7);
    // schedule digest fields (logged; folded lane-parallel when the log fills)
    it_begin(1);
    if (lane == 0) it_put(L, 0, k, ts, T, Np, Cd, blocks, Sp, D, m, nres, nadm, nfin, nrej);
    L.nit += 1;
    it_commit();
    if (!HELP) {
      peak = blocks > peak ? blocks : peak;
      bns += blocks * (u64)T;
    }
    swo_tot += swap_out;
    swi_tot += swap_in;
    if (HELP) {
    } else if (BINNED) {
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
      full_trace_put(fe, tbuf, tcap_b, 1u, ts, te, blocks, flags);
    }
    t = te;
    ++k;
    cyc_normal += (u64)(prof_clock() - clk_a);
  }
  if constexpr (SD) sd_drain();
  else if (!HELP) ev_flush(L);
  u64 dig_s = 0, dig_bh = 0;
  if constexpr (HELP) {  // hand the end time over, wait for the helper's results
    if (lane_id() == 0) {
      ch->t_final = t;
      ch->eprod = L.nev;
      ch->prod = L.nit;
    }
    __threadfence_block();
    __syncwarp();
    if (lane_id() == 0) ch->state = 2u;
    const long long c0 = clock64();
    while (chan_load(&ch->state) != 3u) {
      if (clock64() - c0 > HELPER_TIMEOUT) {
        flags |= TOKENSIM_PT_INTERNAL_ERROR;
        break;
      }
    }
    __threadfence_block();
    dig_s = ch->dig;
    dig_bh = ch->digb;
    bns = ch->bns;
    peak = ch->peak;
    tn = ch->tn;
    fe.n = ch->tn;
    fe.bytes = ch->tb;
    flags |= ch->tflags;
    __syncwarp();
    if (lane_id() == 0) ch->state = 0u;
  } else {
    it_flush(L);
    if (BINNED) {
      while ((i64)bin * W < t) flush_bin();
    }
    dig_s = warp_sum64(L.dig_s);
  }
  // unfinished requests still in R u Q: first-token latency and preemption count
  #pragma unroll 1
  for (u32 x = lane; x < nR + nQ; x += 32) {
    const u32 id = S.id[x];
    write_record(rec + id, S.ttft[x], 0, 0, S.info[x] >> 16, TOKENSIM_REQ_UNFINISHED, 0);
  }
  const u64 dig_b = HELP ? dig_bh : warp_sum64(SD ? sd_dgb : L.dig_b);
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
    st.req_d = 0;  // computed from the records by summary_kernel
    st.total_blocks = total;
    st.peak_blocks = peak;
    st.block_ns_sum = bns;
    st.trace_n[0] = FULLT ? fe.n : min(tn, P.trace_cap);
    for (int q = 1; q < 8; ++q) st.trace_n[q] = 0;
    st.trace_b[0] = FULLT ? fe.bytes : 0;
    for (int q = 1; q < 8; ++q) st.trace_b[q] = 0;
    st.iter_n = min(k, P.it_cap);
    st.n_transfers = 0;
    st.transfer_bytes = 0;
    st.ff_iters = ff_iters;
    st.ff_runs = ff_runs;
    st.cycles = (u64)(clock64() - clk0);
    st.cyc_ff = cyc_ff;
    st.cyc_ff_fail = cyc_ff_fail;
    st.cyc_normal = cyc_normal;
    for (int q = 0; q < 8; ++q) st.phase[q] = ph[q];
    for (int q = 0; q < 8; ++q) st.nphase[q] = nph[q];
    st.n_req = MRM ? mr.ntot : n;
    for (int q = 0; q < 5; ++q) st.ff_fail[q] = ffr[q];
    for (int q = 0; q < 5; ++q) st.ff_cut[q] = ffc[q];
    P.stats[j] = st;
  }
  __syncwarp();
}

// The helper warp of the one-warp-per-SM lean kernel: for each point the simulating warp runs,
// consume its iteration-log ring 32 entries at a time (lane = entry) and produce what the
// simulating warp would otherwise compute on its chain (see HelperChan).
template <int CAP, bool P2>
static __device__ void helper_loop(const SweepParams &P, volatile HelperChan *ch, u32 gwarp, u32 *hbm, u32 *fl) {
  const u32 lane = lane_id();
  const ulonglong2 *ring = P.itlog + (size_t)gwarp * ITCAP * 4;
  const uint4 *evr = P.evlog + (size_t)gwarp * EVCAP;
  u32 *bt = P.bt + (size_t)gwarp * P.bt_tables * CAP * P.bt_len;
  const u32 btl = P.bt_len;
  const bool BINNED = P.trace_mode == TOKENSIM_TRACE_BINNED;
  const bool FULLT = P.trace_mode == TOKENSIM_TRACE_FULL;
  const i64 W = (i64)P.bin_ns;
  while (true) {
    u32 st;
    // 1: a point is running; 2: a short point already finished before we looked; 4: exit.
    // No timeout here: the simulating warp always ends with state 4, and leaving early would
    // turn every later point of this CTA into a timed-out wait.  The waits inside a
    // point keep their bound and flag that point instead.
    while ((st = chan_load(&ch->state)) != 1u && st != 2u && st != 4u) {
    }
    if (st == 4u) return;
    __threadfence_block();
    const u64 j = ch->j;
    // the point's free-block bitmap, replayed from the block events (lowest free first)
    const u64 point = P.begin + j * P.stride;
    const Coords cd = decode_point(point, P.n_pol, P.n_rates, P.n_seeds);
    const DevHP HP = P.hp[(size_t)cd.hw * P.n_pol + cd.pol];
    const u32 nwords = HP.nwords;
    {
      const u32 full_words = (u32)(HP.total_blocks >> 5), tail = (u32)(HP.total_blocks & 31);
      #pragma unroll 1
      for (u32 w = lane; w < nwords; w += 32)
        hbm[w] = w < full_words ? 0xffffffffu : (w == full_words && tail ? ((1u << tail) - 1u) : 0u);
      __syncwarp();
    }
    u32 hint = 0, econs = 0;
    u64 dgb = 0;
    tokensim_mem_sample *trc = P.trace + (size_t)j * P.trace_nw * P.trace_cap;
    FullEnc fe = {0, 0, 0, 0, 0, 0};
    tokensim_iter_record *itr = P.itrec + (size_t)j * P.it_cap;
    u64 dg = 0, bns = 0, peak = 0, tn = 0, bin = 0, acc_bns = 0;
    u32 tflags = 0, acc_max = 0, acc_nit = 0, cons = 0;
    i64 bin_end = W;
    auto flush_bin = [&]() {
      if (tn < P.trace_cap) {
        if (lane == 0) {
          tokensim_mem_sample sm;
          sm.t_ns = (i64)bin * W;
          sm.dur_ns = W;
          sm.block_ns = acc_bns;
          sm.blocks_max = acc_max;
          sm.n_iter = acc_nit;
          trc[tn] = sm;
        }
      } else {
        tflags |= TOKENSIM_PT_TRACE_OVERFLOW;
      }
      ++tn;
      ++bin;
      bin_end += W;
      acc_bns = 0;
      acc_max = 0;
      acc_nit = 0;
    };
    long long c0 = clock64();
    while (true) {
      const u32 s2 = chan_load(&ch->state);  // the state before the producer counts
      __threadfence_block();
      const u32 prod = chan_load(&ch->prod);
      const u32 eprod = chan_load(&ch->eprod);
      __threadfence_block();
      const bool ev_err = !replay_block_events(evr, econs, eprod, hbm, fl, hint, nwords, bt, btl, dgb);
      if (ev_err) tflags |= TOKENSIM_PT_INTERNAL_ERROR;
      __syncwarp();
      if (lane == 0) ch->econs = econs;
      if (prod != cons) {
        #pragma unroll 1
        for (u32 e0 = cons; e0 != prod;) {
          const u32 m = min(32u, prod - e0);
          const bool v = lane < m;
          const u32 e = e0 + lane;
          u64 k = 0, Np = 0, Cd = 0, blocks = 0, w6 = 0, w7 = 0;
          i64 ts = 0, T = 0;
          if (v) {
            const ulonglong2 *q = ring + 4 * (size_t)(e & (ITCAP - 1));
            const ulonglong2 a = q[0], b = q[1], c = q[2], d = q[3];
            k = a.x;
            ts = (i64)a.y;
            T = (i64)b.x;
            Np = b.y;
            Cd = c.x;
            blocks = c.y;
            w6 = d.x;
            w7 = d.y;
            dg += sched_fold(k, ts, T, Np, Cd, blocks, w6, w7);
            if (e < P.it_cap) {
              tokensim_iter_record ir;
              ir.k = k & ((1ull << 40) - 1);
              ir.t_start_ns = ts;
              ir.T_ns = T;
              ir.n_prefill = (u32)(w6 & 0xffff);
              ir.n_decode = (u32)((w6 >> 16) & 0xffff);
              ir.N_p = Np;
              ir.C_d = Cd;
              ir.n_preempted = (u32)((w6 >> 32) & 0xffff);
              ir.n_resumed = (u32)(w6 >> 48);
              ir.n_admitted = (u32)(w7 & 0xffff);
              ir.n_rejected = (u32)(w7 >> 32);
              ir.n_finished = (u32)((w7 >> 16) & 0xffff);
              ir.blocks_in_use = (u32)blocks;
              ir.worker = (u32)(k >> 40);
              ir.pad = 0;
              itr[e] = ir;
            }
            bns += blocks * (u64)T;
            peak = blocks > peak ? blocks : peak;
          }
          const i64 te = ts + T;
          if (BINNED) {  // the stretch's lane-parallel bin walk (reading R5)
            const i64 tend = __shfl_sync(FULLMASK, te, m - 1), tsl = __shfl_sync(FULLMASK, ts, m - 1);
            while (true) {
              const i64 bstart = bin_end - W;
              i64 ov = 0;
              bool cnt_here = false;
              if (v) {
                const i64 lo = ts > bstart ? ts : bstart;
                const i64 hi = te < bin_end ? te : bin_end;
                ov = hi - lo;
                cnt_here = ts >= bstart && ts < bin_end;
              }
              acc_bns += warp_sum64(ov > 0 ? blocks * (u64)ov : 0ull);
              acc_max = max(acc_max, __reduce_max_sync(FULLMASK, ov > 0 ? (u32)blocks : 0u));
              acc_nit += __popc(__ballot_sync(FULLMASK, cnt_here));
              if (tend > bin_end || tsl >= bin_end) flush_bin();
              else break;
            }
          } else if (FULLT) {
            full_trace_put(fe, reinterpret_cast<unsigned char *>(trc), P.trace_cap * sizeof(tokensim_mem_sample), m,
                           ts, te, blocks, tflags);
          }
          e0 += m;
        }
        cons = prod;
        __syncwarp();
        if (lane == 0) ch->cons = cons;
        c0 = clock64();
      } else if (s2 == 2u && econs == eprod) {
        break;
      } else if (clock64() - c0 > HELPER_TIMEOUT) {
        tflags |= TOKENSIM_PT_INTERNAL_ERROR;
        break;
      }
    }
    __threadfence_block();
    if (BINNED) {
      const i64 tf = ch->t_final;
      while ((i64)bin * W < tf) flush_bin();
    }
    const u64 dig = warp_sum64(dg), bsum = warp_sum64(bns);
    u64 pk = peak;
#pragma unroll
    for (u32 o = 16; o; o >>= 1) {
      const u64 y = __shfl_xor_sync(FULLMASK, pk, o);
      pk = y > pk ? y : pk;
    }
    const u64 digb = warp_sum64(dgb);
    if (lane == 0) {
      ch->dig = dig;
      ch->digb = digb;
      ch->bns = bsum;
      ch->peak = pk;
      ch->tn = FULLT ? fe.n : tn;
      ch->tb = fe.bytes;
      ch->tflags = tflags;
    }
    __threadfence_block();
    __syncwarp();
    if (lane == 0) ch->state = 3u;
  }
}

// V: 0 = lean unified (MIXED), 1 = full unified, 2 = 1P:1D pair, 4 = the lean one with compact
// helpers (sim_base_c.cu; sweeps that run several warps per SM), 5 = lean with the helper warp
// and no extended stretches (the xP:yD node, variant 3, is sim_node_kernel: one CTA per point).
// One kernel per variant: its registers and instruction footprint are those of the code it can run.
template <int CAP, int V, bool P2>
__global__ void __launch_bounds__(128, 2) sim_kernel(SweepParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const u32 lane = lane_id(), wib = threadIdx.x >> 5;
  constexpr bool HELPK = (V == 0 || V == 5 || V == 6) && TS_HELPER_WARP;  // one simulating warp + its helper per CTA
  constexpr bool pd = V == 2;  // (the xP:yD node has a kernel of its own: sim_node_kernel, sim_pdn.cuh)
  const size_t base = smem_per_warp_bytes(CAP, P.nwords_max);
  const size_t per_warp = base + (pd ? smem_pd_extra(CAP, P.nwords_max) : 0);
  volatile HelperChan *ch = nullptr;
  if constexpr (HELPK) {
    unsigned char *hb = smem_raw + ((per_warp + 15) & ~(size_t)15);
    ch = reinterpret_cast<volatile HelperChan *>(hb);
    if (threadIdx.x == 0) {  // shared memory starts as garbage: set before either warp looks
      ch->state = 0u;
      ch->eprod = 0u;
      ch->econs = 0u;
    }
    __syncthreads();
    if (wib == 1) {
      u32 *hbm = reinterpret_cast<u32 *>(hb + sizeof(HelperChan));
      helper_loop<CAP, P2>(P, ch, blockIdx.x, hbm, hbm + P.nwords_max);
      return;
    }
  }
  const WarpSmem S = carve(smem_raw + (HELPK ? 0 : wib) * per_warp, CAP);
  const u32 gwarp = HELPK ? blockIdx.x : blockIdx.x * (blockDim.x >> 5) + wib;
  u32 *bt = P.bt + (size_t)gwarp * P.bt_tables * CAP * P.bt_len;
  // Heads (variant 0, strong scaling): the n_heads longest-estimated points each run on an SM
  // of their own -- the first CTA to arrive on an SM takes a head ticket, and the other CTAs on
  // a head's SM leave at once, so the longest serial chains run at their alone speed while the
  // rest of the queue is shared by the other SMs.  Every queue position is claimed exactly once
  // (head positions by atomicCAS on their claim word), so no point is lost or repeated.
  u32 head_qi = 0xffffffffu;
  bool leave = false;
  if constexpr (HELPK) {
    const u32 NH = P.n_heads;
    if (NH) {
      u32 h = 0xffffffffu, lv = 0;
      if (lane == 0) {
        u32 smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        smid &= 255u;
        u32 *cnt = P.sched, *state = P.sched + 256, *ticket = P.sched + 512, *claim = P.sched + 513;
        if (atomicAdd(&cnt[smid], 1u) == 0u) {  // first CTA on this SM
          while (true) {
            const u32 t = atomicAdd(ticket, 1u);
            if (t >= NH) break;
            if (atomicCAS(&claim[t], 0u, 1u) == 0u) {
              h = t;
              break;
            }
          }
          atomicExch(&state[smid], h != 0xffffffffu ? 2u : 1u);
        } else {
          u32 f;
          while ((f = atomicAdd(&state[smid], 0u)) == 0u) {
          }
          lv = f == 2u;
        }
      }
      head_qi = __shfl_sync(FULLMASK, h, 0);
      leave = __shfl_sync(FULLMASK, lv, 0) != 0u;
    }
  }
  while (!leave) {
    u32 qi = 0;
    if (head_qi != 0xffffffffu) {
      qi = head_qi;
      head_qi = 0xffffffffu;
    } else {
      if (lane == 0) {
        if constexpr (HELPK) {
          const u32 NH = P.n_heads;
          qi = NH + atomicAdd(P.queue, 1u);
          if (NH && (u64)qi >= P.n_run) {  // leftovers: head positions no first CTA claimed
            qi = 0xffffffffu;
            u32 *claim = P.sched + 513;
            for (u32 t = 0; t < NH; ++t)
              if (atomicCAS(&claim[t], 0u, 1u) == 0u) {
                qi = t;
                break;
              }
          }
        } else {
          qi = atomicAdd(P.queue, 1u);
        }
      }
      qi = __shfl_sync(FULLMASK, qi, 0);
    }
    if ((u64)qi >= P.n_run) break;
    const u64 j = P.order[qi];
    if constexpr (HELPK) {  // hand the point to the helper
      if (lane == 0) {
        ch->prod = 0u;
        ch->cons = 0u;
        ch->eprod = 0u;
        ch->econs = 0u;
        ch->j = j;
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) ch->state = 1u;
    }
    if constexpr (V == 2) simulate_pd<CAP, P2>(P, j, S, smem_raw + wib * per_warp + base, bt);
    else simulate_unified<CAP, V == 1 || V == 6, P2>(P, j, S, bt, ch);  // V 4: the lean one built with TS_COMPACT
  }
  if constexpr (HELPK) {
    __threadfence_block();
    __syncwarp();
    if (lane == 0) ch->state = 4u;
  }
}

// launch / occupancy helpers for one variant (instantiated by sim_base.cu, sim_base_n.cu,
// sim_base_c.cu, sim_full.cu, sim_pair.cu; the node's are in sim_node.cu)
// V 0 with the helper warp: one simulating warp (wpb = 1) + the helper, and the hand-over
// counters after the warp's shared memory
template <int V>
static __host__ __forceinline__ int sim_threads(int wpb) { return ((V == 0 || V == 5 || V == 6) && TS_HELPER_WARP) ? 64 : wpb * 32; }
// the helper's area: hand-over counters, its replayed bitmap (nwords_max words), 256 extraction slots
static_assert(sizeof(HelperChan) <= kHelperChanBytes, "helper area (ts_internal.cuh)");
template <int V>
static __host__ __forceinline__ size_t sim_smem(size_t smem, u32 nwords_max) {
  return ((V == 0 || V == 5 || V == 6) && TS_HELPER_WARP) ? helper_cta_smem(smem, nwords_max) : smem;
}
template <int CAP, int V, bool P2>
static cudaError_t launch_sim_t(const SweepParams &p, int wpb, int blocks, size_t smem, cudaStream_t st) {
  if ((V == 0 || V == 5 || V == 6) && TS_HELPER_WARP && wpb != 1) return cudaErrorInvalidValue;
  smem = sim_smem<V>(smem, p.nwords_max);
  cudaError_t e = cudaFuncSetAttribute(sim_kernel<CAP, V, P2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  sim_kernel<CAP, V, P2><<<blocks, sim_threads<V>(wpb), smem, st>>>(p);
  return cudaGetLastError();
}
template <int CAP, int V, bool P2>
static cudaError_t occ_t(int wpb, size_t smem, u32 nwords_max, int *b) {
  smem = sim_smem<V>(smem, nwords_max);
  cudaError_t e = cudaFuncSetAttribute(sim_kernel<CAP, V, P2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(b, sim_kernel<CAP, V, P2>, sim_threads<V>(wpb), smem);
}
template <int V, bool P2>
static cudaError_t launch_sim_c(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  switch (cap) {
    case 32: return launch_sim_t<32, V, P2>(p, wpb, blocks, smem, st);
    case 256: return launch_sim_t<256, V, P2>(p, wpb, blocks, smem, st);
    case 1024: return launch_sim_t<1024, V, P2>(p, wpb, blocks, smem, st);
    default: return cudaErrorInvalidValue;
  }
}
template <int V>
static cudaError_t launch_sim_v(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  return p.all_p2 ? launch_sim_c<V, true>(p, cap, wpb, blocks, smem, st)
                  : launch_sim_c<V, false>(p, cap, wpb, blocks, smem, st);
}
template <int V, bool P2>
static cudaError_t sim_occupancy_c(int cap, int wpb, size_t smem, u32 nw, int *b) {
  switch (cap) {
    case 32: return occ_t<32, V, P2>(wpb, smem, nw, b);
    case 256: return occ_t<256, V, P2>(wpb, smem, nw, b);
    case 1024: return occ_t<1024, V, P2>(wpb, smem, nw, b);
    default: return cudaErrorInvalidValue;
  }
}
template <int V>
static cudaError_t sim_occupancy_v(int cap, int wpb, size_t smem, u32 nw, int *b) {
  int b1 = 0, b2 = 0;  // the same resources either way; take the smaller to be safe
  cudaError_t e = sim_occupancy_c<V, true>(cap, wpb, smem, nw, &b1);
  if (e != cudaSuccess) return e;
  e = sim_occupancy_c<V, false>(cap, wpb, smem, nw, &b2);
  *b = b1 < b2 ? b1 : b2;
  return e;
}

}  // namespace ts
