// alu_peak.cu -- measured INT32 ALU and warp-issue peaks of this B200 (VERDICT r1 "Next round #8").
//
// The simulation kernel's roofline is "alu" (nothing is a dense contraction or
// HBM-bound), so its denominator must be a measured integer-ALU throughput, not a nominal one.
//
// Kernel: every thread runs 8 independent dependency chains of 32-bit integer operations in an
// unrolled loop (no memory traffic inside), at full occupancy on every SM.
//   add:  x_i = x_i + y_i  (IADD3 with a zero operand)    -> INT32 add lane-ops/s
//   lop:  x_i = x_i ^ y_i  (LOP3)                          -> logic lane-ops/s
//   mix:  x_i = (x_i + y_i) ^ (x_i >> 3) (IADD3/SHF/LOP3)  -> a simulator-like mix
// Reported per kind: lane-ops/s and warp-instructions/s (SASS instructions of the loop body per
// iteration, counted with cuobjdump by tools/alu_peak.py), best of 5 launches, CUDA events.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peak tools/alu_peak.cu && ./alu_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void __launch_bounds__(1024) alu_kernel(unsigned *out, unsigned seed, int iters) {
  unsigned x0 = seed ^ threadIdx.x, x1 = x0 * 3u, x2 = x0 * 5u, x3 = x0 * 7u, x4 = x0 * 11u, x5 = x0 * 13u,
           x6 = x0 * 17u, x7 = x0 * 19u;
  const unsigned y = seed * 2654435761u + blockIdx.x;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (KIND == 0) {
        asm volatile("add.u32 %0, %0, %8;\n\tadd.u32 %1, %1, %8;\n\tadd.u32 %2, %2, %8;\n\tadd.u32 %3, %3, %8;\n\t"
                     "add.u32 %4, %4, %8;\n\tadd.u32 %5, %5, %8;\n\tadd.u32 %6, %6, %8;\n\tadd.u32 %7, %7, %8;"
                     : "+r"(x0), "+r"(x1), "+r"(x2), "+r"(x3), "+r"(x4), "+r"(x5), "+r"(x6), "+r"(x7)
                     : "r"(y));
      } else if (KIND == 1) {
        // x_i ^= x_{i+1}: a rotating dependency the compiler cannot cancel (x ^ y ^ y = x)
        asm volatile("xor.b32 %0, %0, %1;\n\txor.b32 %1, %1, %2;\n\txor.b32 %2, %2, %3;\n\txor.b32 %3, %3, %4;\n\t"
                     "xor.b32 %4, %4, %5;\n\txor.b32 %5, %5, %6;\n\txor.b32 %6, %6, %7;\n\txor.b32 %7, %7, %8;"
                     : "+r"(x0), "+r"(x1), "+r"(x2), "+r"(x3), "+r"(x4), "+r"(x5), "+r"(x6), "+r"(x7)
                     : "r"(y));
      } else {
        x0 = (x0 + y) ^ (x0 >> 3); x1 = (x1 + y) ^ (x1 >> 3); x2 = (x2 + y) ^ (x2 >> 3); x3 = (x3 + y) ^ (x3 >> 3);
        x4 = (x4 + y) ^ (x4 >> 3); x5 = (x5 + y) ^ (x5 >> 3); x6 = (x6 + y) ^ (x6 >> 3); x7 = (x7 + y) ^ (x7 >> 3);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7;
}

template <int KIND>
static double run(int sms, int iters, double *ms_out) {
  const int threads = 1024, blocks = sms * 2;  // 64 warps per SM (full occupancy)
  unsigned *out;
  cudaMalloc(&out, (size_t)threads * blocks * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  alu_kernel<KIND><<<blocks, threads>>>(out, 1u, iters / 10);  // warm-up
  double best = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    alu_kernel<KIND><<<blocks, threads>>>(out, 12345u + rep, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  *ms_out = best;
  // lane-ops: 8 chains x 16 unrolled x iters per thread (mix counts 3 ops per chain step)
  const double per = 8.0 * 16.0 * iters * (KIND == 2 ? 3.0 : 1.0);
  return per * threads * blocks / (best * 1e-3);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int iters = 20000;
  double ms0, ms1, ms2;
  const double add = run<0>(sms, iters, &ms0), lop = run<1>(sms, iters, &ms1), mix = run<2>(sms, iters, &ms2);
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"iters\": %d, \"add_lane_ops_per_s\": %.6e, \"add_ms\": %.4f, "
         "\"lop_lane_ops_per_s\": %.6e, \"lop_ms\": %.4f, \"mix_lane_ops_per_s\": %.6e, \"mix_ms\": %.4f}\n",
         sms, clk, iters, add, ms0, lop, ms1, mix, ms2);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
