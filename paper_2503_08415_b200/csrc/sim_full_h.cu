// sim_full_h.cu -- the full unified kernel (prefill-first / chunked iterations, multi-round
// conversations + memory cache) with a helper warp per CTA (variant 6), for sweeps with at most
// ~4 points per SM, where each point's serial chain sets the time: block ids, digests and
// traces move to the helper warp as in the lean helper kernel (sim_base.cu), with its extended
// stretches (carried state, up to 64 iterations: c7 -8%, prefill-first / chunked neutral); the
// preload link's pipeline gets a scratch region of its own (the block-event log is the helper's).
#define TS_HELPER_WARP 1
#define TS_XS 1
#define TS_LOGS_BYREF 1
#include "sim_core.cuh"

namespace ts {
cudaError_t launch_sim_full_h(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  return launch_sim_v<6>(p, cap, wpb, blocks, smem, st);
}
cudaError_t sim_occupancy_full_h(int cap, int wpb, size_t smem, u32 nw, int *b) {
  return sim_occupancy_v<6>(cap, wpb, smem, nw, b);
}
}  // namespace ts
