// sim_base_c.cu -- the lean simulation kernel built with compact (out-of-line) helpers, for
// sweeps that put several warps on an SM, where the kernel is instruction-fetch bound.
#define TS_COMPACT 1
#include "sim_core.cuh"

namespace ts {
cudaError_t launch_sim_base_c(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  return launch_sim_v<4>(p, cap, wpb, blocks, smem, st);
}
cudaError_t sim_occupancy_base_c(int cap, int wpb, size_t smem, u32 nw, int *b) {
  return sim_occupancy_v<4>(cap, wpb, smem, nw, b);
}
}  // namespace ts
