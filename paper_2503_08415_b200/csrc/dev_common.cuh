// dev_common.cuh -- warp-level primitives and the c.6 digest mixer shared by the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "ts_internal.cuh"

namespace ts {

#define FULLMASK 0xffffffffu

// Per-path / per-phase cycle counters of the point profile (tokensim_get_point_profile).
// Off in the product build (they cost 5-10% of the simulation kernel); build with
// -DTS_PROFILE=1 (tools/prof_run.py --build) to read them, otherwise they read 0.
#ifndef TS_PROFILE
#define TS_PROFILE 0
#endif
// TS_COMPACT (set by sim_base_c.cu, the lean kernel for sweeps with several warps per SM): small hot helpers are
// compiled out of line, trading a call's latency for a smaller instruction footprint -- at
// 8 warps per SM the kernels are instruction-fetch bound.
#ifndef TS_COMPACT
#define TS_COMPACT 0
#endif
#if TS_COMPACT
#define TS_HELPER static __device__ __noinline__
#else
#define TS_HELPER __device__ __forceinline__
#endif
__device__ __forceinline__ long long prof_clock() {
#if TS_PROFILE
  return clock64();
#else
  return 0;
#endif
}

__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// TS_COMPACT_SCAN (A/B): the warp scan and the 64-bit warp sum out of line as well
#ifndef TS_COMPACT_SCAN
#define TS_COMPACT_SCAN 0
#endif
#if TS_COMPACT_SCAN
#define TS_SCANFN static __device__ __noinline__
#else
#define TS_SCANFN __device__ __forceinline__
#endif
TS_SCANFN u32 scan_incl(u32 x) {
  const u32 l = lane_id();
#pragma unroll
  for (u32 o = 1; o < 32; o <<= 1) {
    u32 y = __shfl_up_sync(FULLMASK, x, o);
    if (l >= o) x += y;
  }
  return x;
}
// Exact wrapping 64-bit warp sum with three 32-bit REDUX ops: split into 21/21/22-bit
// digits (each digit sum over 32 lanes stays below 2^27) and recombine mod 2^64.
TS_SCANFN u64 warp_sum64(u64 x) {
  const u32 a = __reduce_add_sync(FULLMASK, (u32)(x & 0x1FFFFFull));
  const u32 b = __reduce_add_sync(FULLMASK, (u32)((x >> 21) & 0x1FFFFFull));
  const u32 c = __reduce_add_sync(FULLMASK, (u32)(x >> 42));
  return (u64)a + ((u64)b << 21) + ((u64)c << 42);
}
__device__ __forceinline__ u64 shfl64(u64 x, u32 src) { return __shfl_sync(FULLMASK, x, src); }
__device__ __forceinline__ i64 shfl64i(i64 x, u32 src) { return __shfl_sync(FULLMASK, x, src); }

// r-th (0-based) set bit of w (r < popc(w))
TS_HELPER u32 select_bit(u32 w, u32 r) {
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
// block event (k, kind, id, block) -> fold(k | kind << 48, id | block << 32)
__device__ __forceinline__ u64 fold_event(u32 k, u32 kind, u32 id, u32 blk) {
  u64 h = FOLD_INIT;
  h = mix64(h ^ ((u64)k | ((u64)kind << 48)));
  h = mix64(h ^ ((u64)id | ((u64)blk << 32)));
  return h;
}

// block size arithmetic: shifts/masks when block_size is a power of two (the common case)
struct BSz {
  u32 bs, sh, mask;
  bool p2;
  __device__ __forceinline__ u32 div(u32 x) const { return p2 ? (x >> sh) : x / bs; }
  __device__ __forceinline__ u32 mod(u32 x) const { return p2 ? (x & mask) : x % bs; }
  __device__ __forceinline__ u32 cdiv(u32 x) const { return p2 ? ((x + mask) >> sh) : (x + bs - 1) / bs; }
};

}  // namespace ts
