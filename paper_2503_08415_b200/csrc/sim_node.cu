// sim_node.cu -- the xP:yD node kernel with a global scheduler (NEXT-1, sim_pdn.cuh): one CTA of
// y warps per point (warp j: decode worker j; warp 0 also the scheduler and the prefill workers).
#define TS_LOGS_BYREF 1
#include "sim_core.cuh"

namespace ts {
template <int CAP, bool P2, bool TWO, bool SW>
static cudaError_t launch_node_k(const SweepParams &p, int blocks, size_t smem, cudaStream_t st) {
  cudaError_t e =
      cudaFuncSetAttribute(sim_node_kernel<CAP, P2, TWO, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  sim_node_kernel<CAP, P2, TWO, SW><<<blocks, ((int)p.pd_y + (SW ? 1 : 0)) * 32, smem, st>>>(p);
  return cudaGetLastError();
}
template <int CAP, bool P2>
static cudaError_t launch_node_t(const SweepParams &p, int blocks, size_t smem, cudaStream_t st) {
  if (p.node_two) return launch_node_k<CAP, P2, true, false>(p, blocks, smem, st);
  return p.node_sw ? launch_node_k<CAP, P2, false, true>(p, blocks, smem, st)
                   : launch_node_k<CAP, P2, false, false>(p, blocks, smem, st);
}
template <int CAP, bool P2, bool TWO, bool SW>
static cudaError_t occ_node_k(int warps, size_t smem, int *b) {
  cudaError_t e =
      cudaFuncSetAttribute(sim_node_kernel<CAP, P2, TWO, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(b, sim_node_kernel<CAP, P2, TWO, SW>, warps * 32, smem);
}
// warps: the CTA's warps (bits 0-3), + 16 for the two-CTAs-per-SM build, + 32 for the
// scheduler-warp build
template <int CAP, bool P2>
static cudaError_t occ_node_t(int warps, size_t smem, int *b) {
  const int w = warps & 15;
  if (warps & 16) return occ_node_k<CAP, P2, true, false>(w, smem, b);
  return (warps & 32) ? occ_node_k<CAP, P2, false, true>(w, smem, b) : occ_node_k<CAP, P2, false, false>(w, smem, b);
}
template <bool P2>
static cudaError_t launch_node_c(const SweepParams &p, int cap, int blocks, size_t smem, cudaStream_t st) {
  switch (cap) {
    case 32: return launch_node_t<32, P2>(p, blocks, smem, st);
    case 256: return launch_node_t<256, P2>(p, blocks, smem, st);
    case 1024: return launch_node_t<1024, P2>(p, blocks, smem, st);
    default: return cudaErrorInvalidValue;
  }
}
template <bool P2>
static cudaError_t occ_node_c(int cap, int warps, size_t smem, int *b) {
  switch (cap) {
    case 32: return occ_node_t<32, P2>(warps, smem, b);
    case 256: return occ_node_t<256, P2>(warps, smem, b);
    case 1024: return occ_node_t<1024, P2>(warps, smem, b);
    default: return cudaErrorInvalidValue;
  }
}
// (wpb is ignored: a node CTA has pd_y (+1 with the scheduler warp) warps and holds one point)
cudaError_t launch_sim_node(const SweepParams &p, int cap, int wpb, int blocks, size_t smem, cudaStream_t st) {
  (void)wpb;
  return p.all_p2 ? launch_node_c<true>(p, cap, blocks, smem, st) : launch_node_c<false>(p, cap, blocks, smem, st);
}
// warps: see occ_node_t
cudaError_t sim_occupancy_node(int cap, int warps, size_t smem, u32 nw, int *b) {
  (void)nw;
  int b1 = 0, b2 = 0;
  cudaError_t e = occ_node_c<true>(cap, warps, smem, &b1);
  if (e != cudaSuccess) return e;
  e = occ_node_c<false>(cap, warps, smem, &b2);
  *b = b1 < b2 ? b1 : b2;
  return e;
}
}  // namespace ts
