// Microbenchmark (tool, not product): FP64 tensor-core MMA (mma.sync m8n8k4
// f64) throughput on B200 vs the DFMA peak, operands from registers or
// shared memory.
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// ACC independent accumulator tiles per warp (ILP), W warps per CTA
template <int ACC, int SMEM>
__global__ void __launch_bounds__(256, 1) dmma_kernel(double* out, int iters) {
  __shared__ double sa[32 * 64], sb[32 * 64];
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) { sa[i] = 1e-3 * i; sb[i] = 1e-4 * i; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double d[ACC][2];
#pragma unroll
  for (int k = 0; k < ACC; ++k) d[k][0] = d[k][1] = 0.0;
  double a[4], b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { a[k] = sa[lane + 32 * k]; b[k] = sb[lane + 32 * k]; }
  for (int it = 0; it < iters; ++it) {
    asm volatile("" ::: "memory");
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      double av[4], bv[4];
      if (SMEM) {
#pragma unroll
        for (int k = 0; k < 4; ++k) { av[k] = sa[(kk * 4 + k) * 32 + lane]; bv[k] = sb[(kk * 4 + k) * 32 + lane]; }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) { av[k] = a[k]; bv[k] = b[(k + kk) & 3]; }
      }
      // ACC tiles: tile (i, j) uses a[i % 4], b[j % 4]
#pragma unroll
      for (int k = 0; k < ACC; ++k) dmma(d[k][0], d[k][1], av[k & 3], bv[(k >> 2) & 3]);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < ACC; ++k) s += d[k][0] + d[k][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

extern "C" int mb_dmma(int acc, int smem, int blocks, double* out, int iters, void* st) {
  if (acc == 8 && !smem) dmma_kernel<8, 0><<<blocks, 256, 0, (cudaStream_t)st>>>(out, iters);
  else if (acc == 16 && !smem) dmma_kernel<16, 0><<<blocks, 256, 0, (cudaStream_t)st>>>(out, iters);
  else if (acc == 16 && smem) dmma_kernel<16, 1><<<blocks, 256, 0, (cudaStream_t)st>>>(out, iters);
  else if (acc == 32 && smem) dmma_kernel<32, 1><<<blocks, 256, 0, (cudaStream_t)st>>>(out, iters);
  else if (acc == 32 && !smem) dmma_kernel<32, 0><<<blocks, 256, 0, (cudaStream_t)st>>>(out, iters);
  else return -1;
  return (int)cudaGetLastError();
}
