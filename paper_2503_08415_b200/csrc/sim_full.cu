// sim_full.cu -- the full unified simulation kernel variant: prefill-first and chunked
// iterations (NEXT-3), multi-round conversations + memory cache (NEXT-2), the preload link
// (NEXT-4) (see sim_core.cuh).
#define TS_LOGS_BYREF 1
#include "sim_core.cuh"

namespace ts {
cudaError_t launch_sim_full(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  return launch_sim_v<1>(p, cap, wpb, blocks, smem, st);
}
cudaError_t sim_occupancy_full(int cap, int wpb, size_t smem, u32 nw, int *b) {
  return sim_occupancy_v<1>(cap, wpb, smem, nw, b);
}
}  // namespace ts
