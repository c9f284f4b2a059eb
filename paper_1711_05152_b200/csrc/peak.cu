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

// Random 32-bit operations on an L2-resident bitmap (the alias kernels'
// access pattern, K3): mode 0 atomicOr with the returned value used (the mark
// kernel), mode 1 loads (the mask kernel).  ops per launch = blocks * 256 *
// per_thread.  The K3 roofline denominator (its bytes are L2-resident).
__device__ __forceinline__ uint32_t peak_hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(256) l2_random_peak_kernel(uint32_t* bits, uint32_t words, int per_thread,
                                                             int mode, uint32_t* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
#pragma unroll 8
  for (int i = 0; i < per_thread; ++i) {
    const uint32_t h = peak_hash32(tid * 131u + (uint32_t)i * 7919u);
    const uint32_t w = h % words;
    if (mode == 0) acc |= atomicOr(&bits[w], 1u << (h >> 27));
    else if (mode == 2) atomicAdd(&bits[w], 1u);  // result unused: RED (the alias counter variant)
    else acc |= __ldg(&bits[w]);
  }
  if (acc == 0x12345678u) sink[0] = acc;  // keep the results alive
}

int launch_l2_random_peak(uint32_t* bits, uint32_t words, int blocks, int per_thread, int mode, cudaStream_t st) {
  l2_random_peak_kernel<<<blocks, 256, 0, st>>>(bits, words, per_thread, mode, bits);
  SFFT_CHECK_LAUNCH();
  return 0;
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
