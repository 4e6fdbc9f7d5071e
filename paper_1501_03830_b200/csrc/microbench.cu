// FP64 peak probes: DMMA (mma.sync m8n8k4 f64) and DFMA issue-bound loops.
// Used once per box to fix the FP64 roofline denominator (MEASURED_PEAKS.json
// carries no FP64 figure).
#include "common.cuh"

namespace bse {

__global__ void __launch_bounds__(256) peak_dmma_kernel(int iters, double* sink) {
  double acc[8][2];
  const int lane = threadIdx.x & 31;
  double a = 1.0 + 1e-9 * lane, b = 1.0 - 1e-9 * lane;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma8x8x4(acc[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 123.456) sink[threadIdx.x] = s;  // keep the loop alive
}

__global__ void __launch_bounds__(256) peak_dfma_kernel(int iters, double* sink) {
  double acc[8];
  const double a = 1.0 + 1e-12 * threadIdx.x, b = 0.999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 123.456) sink[threadIdx.x] = s;
}

// Returns flops executed by one launch.
double launch_peak(int which, int blocks, int iters, double* sink, cudaStream_t s) {
  if (which == 0) {
    peak_dmma_kernel<<<blocks, 256, 0, s>>>(iters, sink);
    return 2.0 * 256.0 * 8.0 * iters * (blocks * 256 / 32);
  }
  peak_dfma_kernel<<<blocks, 256, 0, s>>>(iters, sink);
  return 2.0 * 8.0 * iters * (double)blocks * 256;
}

}  // namespace bse
