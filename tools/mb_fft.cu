// Microbenchmark (tool, not product): shared-memory-only cost of the row
// pass's two 4096-point FFTs (no global traffic), 256 threads, 2 CTAs/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC
//        -I paper_1711_05152_b200/csrc -o tools/_mb_fft.so tools/mb_fft.cu
#include "fft.cuh"

using namespace sfft;

template <int MODE>
__global__ void __launch_bounds__(FFT_T, 2) mb_row_kernel(const double2* __restrict__ tw, double2* out, int reps) {
  extern __shared__ double2 s[];
  for (int f = threadIdx.x; f < 4096; f += FFT_T) s[Tile<4096>::pad(f)] = make_double2(1e-3 * f, 1.0);
  __syncthreads();
  // no loop (a loop makes ptxas keep every pass's addresses live and spill)
  block_fft<12, false, 4096>(s, tw);
  if (MODE == 1) {
    for (int f = threadIdx.x; f < 4096; f += FFT_T) s[Tile<4096>::pad(f)] = cmul(s[Tile<4096>::pad(f)], make_double2(0.5, 0.25));
    __syncthreads();
  }
  block_fft<12, true, 4096>(s, tw);
  if (threadIdx.x == 0 && s[0].x == 12345.0) out[blockIdx.x] = s[1];
}

extern "C" int mb_row(int mode, int blocks, const double* tw, double* out, int reps, void* st) {
  const size_t sm = (size_t)Tile<4096>::rstride(4096) * sizeof(double2);
  if (mode == 0) {
    cudaFuncSetAttribute((const void*)mb_row_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    mb_row_kernel<0><<<blocks, FFT_T, sm, (cudaStream_t)st>>>((const double2*)tw, (double2*)out, reps);
  } else {
    cudaFuncSetAttribute((const void*)mb_row_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    mb_row_kernel<1><<<blocks, FFT_T, sm, (cudaStream_t)st>>>((const double2*)tw, (double2*)out, reps);
  }
  return (int)cudaGetLastError();
}
