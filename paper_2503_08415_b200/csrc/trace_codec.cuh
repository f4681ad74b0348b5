// trace_codec.cuh -- the compressed FULL memory-trace writer (SURVEY §8(a.8) "FULL (delta +
// varint)", G5/H6; the memory-footprint-over-time output of P:552-565, one sample per iteration,
// reading A28).
//
// Stream format (per point and worker, little-endian bytes, documented in include/tokensim.h):
// one record per iteration, three unsigned LEB128 varints
//     gap   = t_start_k - t_end_{k-1}          (idle time before the iteration, >= 0)
//     dT    = zigzag(T_k - T_{k-1})            (iteration time delta)
//     dB    = zigzag(blocks_k - blocks_{k-1})  (blocks-in-use delta)
// with t_end_{-1} = T_{-1} = blocks_{-1} = 0.  A decode stretch has gap 0, a dT of a few hundred ns
// per decode and dB in {0, 1, ...}: ~4 B per iteration instead of the 32-B sample.  A record that
// would cross the capacity is not written; the stream then ends (overflow flag) so it always
// decodes to a prefix of whole iterations.
#pragma once
#include "dev_common.cuh"

namespace ts {

struct FullEnc {   // lane-uniform encoder state of one worker's stream
  u64 bytes;       // bytes written
  u64 n;           // records (iterations) written
  i64 te, T;       // previous iteration's end and duration
  u32 blk, ovf;    // previous blocks in use; 1 once the stream is closed by its capacity
};

__device__ __forceinline__ u32 varint_len(u64 x) { return x ? (u32)((70 - __clzll((long long)x)) / 7) : 1u; }
__device__ __forceinline__ u64 zigzag64(i64 v) { return ((u64)v << 1) ^ (u64)(v >> 63); }
__device__ __forceinline__ unsigned char *put_varint(unsigned char *p, u64 x) {
  while (x >= 0x80u) {
    *p++ = (unsigned char)(x | 0x80u);
    x >>= 7;
  }
  *p++ = (unsigned char)x;
  return p;
}

// Warp-cooperative: lanes j < J hold iteration j of a stretch, (ts, te, blocks), in order.
// Lane-uniform callers (one iteration) pass J = 1 with the values on lane 0.
static __device__ __noinline__ void full_trace_put(FullEnc &E, unsigned char *buf, u64 cap, u32 J, i64 ts, i64 te,
                                            u64 blocks, u32 &flags) {
  const u32 lane = lane_id();
  const bool lj = lane < J;
  const i64 T = te - ts;
  i64 pte = __shfl_up_sync(FULLMASK, te, 1), pT = __shfl_up_sync(FULLMASK, T, 1);
  u32 pb = __shfl_up_sync(FULLMASK, (u32)blocks, 1);
  if (lane == 0) {
    pte = E.te;
    pT = E.T;
    pb = E.blk;
  }
  const u64 a = (u64)(ts - pte), b = zigzag64(T - pT), c = zigzag64((i64)(u32)blocks - (i64)pb);
  const u32 len = lj ? varint_len(a) + varint_len(b) + varint_len(c) : 0u;
  const u32 incl = scan_incl(len);
  if (!E.ovf) {
    const bool fits = lj && E.bytes + incl <= cap;
    if (fits) {
      unsigned char *p = buf + E.bytes + (incl - len);
      p = put_varint(p, a);
      p = put_varint(p, b);
      put_varint(p, c);
    }
    const u32 nf = __popc(__ballot_sync(FULLMASK, fits));
    if (nf) E.bytes += __shfl_sync(FULLMASK, incl, nf - 1);
    E.n += nf;
    if (nf < J) E.ovf = 1u;
  }
  if (E.ovf) flags |= TOKENSIM_PT_TRACE_OVERFLOW;
  E.te = __shfl_sync(FULLMASK, te, J - 1);
  E.T = __shfl_sync(FULLMASK, T, J - 1);
  E.blk = __shfl_sync(FULLMASK, (u32)blocks, J - 1);
}

}  // namespace ts
