// Register-resident DFMA loop: the measured FP64 roofline denominator
// (MEASURED_PEAKS.json carries no FP64 figure).
#include "common.cuh"

namespace sfft {

__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double seed) {
  double a[8], b = 1.0000001 + 1e-9 * threadIdx.x, c = 0.9999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], c, -b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;  // keep the loop alive
}

// FP64 tensor-core peak: 16 independent DMMA (m8n8k4 f64) accumulators per
// warp, register operands.  flop per launch = blocks * 8 warps * iters * 16 * 512
__global__ void __launch_bounds__(256) fp64_mma_peak_kernel(double* out, int iters, double seed) {
  double d[16][2];
#pragma unroll
  for (int k = 0; k < 16; ++k) d[k][0] = d[k][1] = 0.0;
  const double a = seed + 1e-9 * threadIdx.x, b = 0.999999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += d[k][0] + d[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;  // keep the loop alive
}

int launch_fp64_mma_peak(double* out, int iters, int blocks, cudaStream_t st) {
  fp64_mma_peak_kernel<<<blocks, 256, 0, st>>>(out, iters, 0.5);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_fp64_peak(double* out, int iters, int blocks, cudaStream_t st) {
  fp64_peak_kernel<<<blocks, 256, 0, st>>>(out, iters, 0.5);
  SFFT_CHECK_LAUNCH();
  return 0;
}

}  // namespace sfft
