// sim_full.cu -- the full simulation kernel variant: chunked prefill (NEXT-3b), multi-round
// conversations + memory cache (NEXT-2), the preload link (NEXT-4), the 1P:1D pair (a.9) and the
// xP:yD node (NEXT-1) (see sim_core.cuh).
#define TS_LOGS_BYREF 1
#include "sim_core.cuh"

namespace ts {
cudaError_t launch_sim_full(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  return launch_sim_v<true>(p, cap, wpb, blocks, smem, st);
}
cudaError_t sim_occupancy_full(int cap, int wpb, size_t smem, int *b) { return sim_occupancy_v<true>(cap, wpb, smem, b); }
}  // namespace ts
