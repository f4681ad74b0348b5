// sim_base.cu -- the lean simulation kernel variant for sweeps with at most one point per SM:
// unified topology, MIXED iterations, generated or traced single-round workloads, and a helper
// warp per CTA (see sim_core.cuh).
#define TS_HELPER_WARP 1  // one simulating warp per SM, plus a helper warp for digests and traces
#include "sim_core.cuh"

namespace ts {
cudaError_t launch_sim_base(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  return launch_sim_v<0>(p, cap, wpb, blocks, smem, st);
}
cudaError_t sim_occupancy_base(int cap, int wpb, size_t smem, u32 nw, int *b) {
  return sim_occupancy_v<0>(cap, wpb, smem, nw, b);
}
size_t sim_smem_per_warp(int cap, u32 nwords_max, bool pd, u32 node_x, u32 node_y) {
  return sim_smem_per_warp_impl(cap, nwords_max, pd, node_x, node_y);
}
}  // namespace ts
