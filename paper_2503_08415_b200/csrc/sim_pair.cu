// sim_pair.cu -- the 1P:1D disaggregated pair kernel variant (a.9, sim_pd.cuh).  Built with
// the compact (out-of-line) helpers: its sweeps (C5: 8,192 pairs per GPU) put 8 warps on an SM,
// where instruction fetch binds (C5 every-8th-point 3542 -> 3449 ms).
#define TS_LOGS_BYREF 1
#define TS_COMPACT 1
#define TS_COMPACT_SCAN 1  // warp scans / 64-bit sums out of line too: C5 -5% (C3's kernel: +10%)

#include "sim_core.cuh"

namespace ts {
cudaError_t launch_sim_pair(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  return launch_sim_v<2>(p, cap, wpb, blocks, smem, st);
}
cudaError_t sim_occupancy_pair(int cap, int wpb, size_t smem, u32 nw, int *b) {
  return sim_occupancy_v<2>(cap, wpb, smem, nw, b);
}
}  // namespace ts
