// sim_base_n.cu -- the helper-warp lean kernel without extended stretches (variant 5), for
// latency-bound sweeps with more than ~2 points per SM: there its larger hot code (carried
// stretch state, 64-iteration stretches) costs more in instruction fetch than it saves
// (DESIGN.md §7-§8).
#define TS_HELPER_WARP 1
#define TS_XS 0
#include "sim_core.cuh"

namespace ts {
cudaError_t launch_sim_base_n(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  return launch_sim_v<5>(p, cap, wpb, blocks, smem, st);
}
cudaError_t sim_occupancy_base_n(int cap, int wpb, size_t smem, u32 nw, int *b) {
  return sim_occupancy_v<5>(cap, wpb, smem, nw, b);
}
}  // namespace ts
