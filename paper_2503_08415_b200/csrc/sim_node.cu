// sim_node.cu -- the xP:yD node kernel variant with a global scheduler (NEXT-1, sim_pdn.cuh).
#define TS_LOGS_BYREF 1
#include "sim_core.cuh"

namespace ts {
cudaError_t launch_sim_node(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  return launch_sim_v<3>(p, cap, wpb, blocks, smem, st);
}
cudaError_t sim_occupancy_node(int cap, int wpb, size_t smem, u32 nw, int *b) {
  return sim_occupancy_v<3>(cap, wpb, smem, nw, b);
}
}  // namespace ts
