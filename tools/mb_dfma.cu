// Microbenchmark (tool, not product): DFMA throughput of complex register
// tiles (TI x TJ complex accumulators per thread) as used by the sampling
// kernel's consumers, at W warps per SM, operands from shared memory (as in
// the kernel) or from registers, plus a real-valued calibration loop with one
// or two non-reused operands per DFMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o tools/_mb_dfma.so tools/mb_dfma.cu
#include <cuda_runtime.h>
#include <cstdint>

// ORDER 0: j outer, i inner, two half passes (the kernel's order)
// ORDER 1: i outer, j inner, two half passes
// ORDER 2: j outer, i inner, all four FMAs of one complex MAC together
template <int W, int SMEM, int TI, int TJ, int ORDER>
__global__ void __launch_bounds__(32 * W, 1) mb_kernel(double* out, int chunks) {
  __shared__ double2 As[16 * 16 * TI];
  __shared__ double2 Bs[16 * 16 * TJ];
  for (int i = threadIdx.x; i < 16 * 16 * TI; i += blockDim.x) As[i] = make_double2(1e-3 * i, 2e-3);
  for (int i = threadIdx.x; i < 16 * 16 * TJ; i += blockDim.x) Bs[i] = make_double2(1e-3, 1e-4 * i);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = lane & 15, ty = ((lane >> 4) + 2 * w) & 15;
  double2 acc[TI][TJ];
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TJ; ++j) acc[i][j] = make_double2(0.0, 0.0);
  double2 ra[TI], rb[TJ];
#pragma unroll
  for (int i = 0; i < TI; ++i) ra[i] = As[tx + 16 * i];
#pragma unroll
  for (int j = 0; j < TJ; ++j) rb[j] = Bs[ty + 16 * j];
  for (int c = 0; c < chunks; ++c) {
    asm volatile("" ::: "memory");  // as the real kernel's barrier: no hoisting of smem loads
    if (ORDER == 4) {
      double2 a[2][TI], b[2][TJ];
#pragma unroll
      for (int i = 0; i < TI; ++i) a[0][i] = As[tx + 16 * i];
#pragma unroll
      for (int j = 0; j < TJ; ++j) b[0][j] = Bs[ty + 16 * j];
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const int cu = kk & 1, nx = cu ^ 1;
        if (kk + 1 < 16) {
#pragma unroll
          for (int i = 0; i < TI; ++i) a[nx][i] = As[(kk + 1) * 16 * TI + tx + 16 * i];
#pragma unroll
          for (int j = 0; j < TJ; ++j) b[nx][j] = Bs[(kk + 1) * 16 * TJ + ty + 16 * j];
        }
#pragma unroll
        for (int i = 0; i < TI; ++i) {
#pragma unroll
          for (int j = 0; j < TJ; ++j) {
            acc[i][j].x = fma(a[cu][i].x, b[cu][j].x, acc[i][j].x);
            acc[i][j].y = fma(a[cu][i].x, b[cu][j].y, acc[i][j].y);
          }
#pragma unroll
          for (int j = 0; j < TJ; ++j) {
            acc[i][j].x = fma(-a[cu][i].y, b[cu][j].y, acc[i][j].x);
            acc[i][j].y = fma(a[cu][i].y, b[cu][j].x, acc[i][j].y);
          }
        }
      }
      continue;
    }
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double2 a[TI], b[TJ];
      if (SMEM) {
#pragma unroll
        for (int i = 0; i < TI; ++i) a[i] = As[kk * 16 * TI + tx + 16 * i];
#pragma unroll
        for (int j = 0; j < TJ; ++j) b[j] = Bs[kk * 16 * TJ + ty + 16 * j];
      } else {
#pragma unroll
        for (int i = 0; i < TI; ++i) a[i] = ra[i];  // no reassociation: the FMAs stay
#pragma unroll
        for (int j = 0; j < TJ; ++j) b[j] = rb[(j + kk) % TJ];
      }
      if (ORDER == 0) {
#pragma unroll
        for (int j = 0; j < TJ; ++j) {
#pragma unroll
          for (int i = 0; i < TI; ++i) {
            acc[i][j].x = fma(a[i].x, b[j].x, acc[i][j].x);
            acc[i][j].y = fma(a[i].x, b[j].y, acc[i][j].y);
          }
#pragma unroll
          for (int i = 0; i < TI; ++i) {
            acc[i][j].x = fma(-a[i].y, b[j].y, acc[i][j].x);
            acc[i][j].y = fma(a[i].y, b[j].x, acc[i][j].y);
          }
        }
      } else if (ORDER == 1) {
#pragma unroll
        for (int i = 0; i < TI; ++i) {
#pragma unroll
          for (int j = 0; j < TJ; ++j) {
            acc[i][j].x = fma(a[i].x, b[j].x, acc[i][j].x);
            acc[i][j].y = fma(a[i].x, b[j].y, acc[i][j].y);
          }
#pragma unroll
          for (int j = 0; j < TJ; ++j) {
            acc[i][j].x = fma(-a[i].y, b[j].y, acc[i][j].x);
            acc[i][j].y = fma(a[i].y, b[j].x, acc[i][j].y);
          }
        }
      } else if (ORDER == 3) {
        // snake: every DFMA shares one multiplicand (same operand slot) with the previous one
#pragma unroll
        for (int i = 0; i < TI; ++i) {
#pragma unroll
          for (int jj = 0; jj < TJ; ++jj) {
            const int j = jj;
            if ((i & 1) == 0) {
              acc[i][j].x = fma(b[j].x, a[i].x, acc[i][j].x);
              acc[i][j].y = fma(b[j].y, a[i].x, acc[i][j].y);
            } else {
              acc[i][j].y = fma(b[j].y, a[i].x, acc[i][j].y);
              acc[i][j].x = fma(b[j].x, a[i].x, acc[i][j].x);
            }
          }
#pragma unroll
          for (int jj = 0; jj < TJ; ++jj) {
            const int j = TJ - 1 - jj;
            if ((i & 1) == 0) {
              acc[i][j].y = fma(b[j].x, a[i].y, acc[i][j].y);
              acc[i][j].x = fma(-b[j].y, a[i].y, acc[i][j].x);
            } else {
              acc[i][j].x = fma(-b[j].y, a[i].y, acc[i][j].x);
              acc[i][j].y = fma(b[j].x, a[i].y, acc[i][j].y);
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < TJ; ++j)
#pragma unroll
          for (int i = 0; i < TI; ++i) {
            acc[i][j].x = fma(a[i].x, b[j].x, acc[i][j].x);
            acc[i][j].x = fma(-a[i].y, b[j].y, acc[i][j].x);
            acc[i][j].y = fma(a[i].x, b[j].y, acc[i][j].y);
            acc[i][j].y = fma(a[i].y, b[j].x, acc[i][j].y);
          }
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TJ; ++j) s += acc[i][j].x + acc[i][j].y;
  if (s == 1234.5) out[threadIdx.x] = s;
}

// calibration: 16 independent chains, FRESH = 1: a = fma(a, b, c) (b, c shared),
// FRESH = 2: a_i = fma(a_i, b_i, c) (distinct b_i per chain)
template <int FRESH>
__global__ void __launch_bounds__(256) cal_kernel(double* out, int iters) {
  double a[16], b[16];
  const double c = 0.9999999;
#pragma unroll
  for (int i = 0; i < 16; ++i) { a[i] = 0.5 + i; b[i] = 1.0000001 + 1e-9 * (threadIdx.x + i); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], FRESH == 2 ? b[i] : b[0], c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

#define MB_CASE(ID, W, S, TI, TJ, O)                                                  \
  if (id == ID) {                                                                     \
    mb_kernel<W, S, TI, TJ, O><<<blocks, 32 * W, 0, (cudaStream_t)st>>>(out, chunks); \
    return (int)cudaGetLastError();                                                   \
  }

// returns -1 for an unknown id; flops per launch = blocks*32*W*chunks*16*TI*TJ*8
extern "C" int mb_run(int id, int blocks, double* out, int chunks, void* st) {
  MB_CASE(0, 8, 1, 4, 8, 0) MB_CASE(1, 8, 0, 4, 8, 0)
  MB_CASE(2, 8, 1, 4, 8, 1) MB_CASE(3, 8, 0, 4, 8, 1)
  MB_CASE(4, 8, 1, 4, 8, 2) MB_CASE(5, 8, 0, 4, 8, 2)
  MB_CASE(6, 8, 1, 8, 4, 0) MB_CASE(7, 8, 0, 8, 4, 0)
  MB_CASE(8, 8, 1, 8, 4, 1) MB_CASE(9, 8, 0, 8, 4, 1)
  MB_CASE(10, 16, 1, 4, 4, 0) MB_CASE(11, 16, 0, 4, 4, 0)
  MB_CASE(12, 12, 1, 4, 4, 0) MB_CASE(13, 12, 0, 4, 4, 0)
  MB_CASE(14, 8, 1, 4, 8, 3) MB_CASE(15, 8, 0, 4, 8, 3)
  MB_CASE(16, 8, 1, 8, 4, 3) MB_CASE(17, 8, 0, 8, 4, 3)
  MB_CASE(18, 8, 1, 4, 8, 4) MB_CASE(19, 4, 1, 4, 8, 1)
  if (id == 100) { cal_kernel<1><<<blocks, 256, 0, (cudaStream_t)st>>>(out, chunks); return (int)cudaGetLastError(); }
  if (id == 101) { cal_kernel<2><<<blocks, 256, 0, (cudaStream_t)st>>>(out, chunks); return (int)cudaGetLastError(); }
  return -1;
}

extern "C" int mb_info(int id, int* w, int* ti, int* tj) {
  const int tab[20][3] = {{8, 4, 8}, {8, 4, 8}, {8, 4, 8}, {8, 4, 8}, {8, 4, 8}, {8, 4, 8}, {8, 8, 4}, {8, 8, 4},
                          {8, 8, 4}, {8, 8, 4}, {16, 4, 4}, {16, 4, 4}, {12, 4, 4}, {12, 4, 4}, {8, 4, 8}, {8, 4, 8}, {8, 8, 4}, {8, 8, 4}, {8, 4, 8}, {4, 4, 8}};
  if (id < 0 || id >= 20) return -1;
  *w = tab[id][0]; *ti = tab[id][1]; *tj = tab[id][2];
  return 0;
}

// launch cost vs kernel-parameter size (host time per launch)
template <int BYTES>
struct Blob { char b[BYTES]; };
template <int BYTES>
__global__ void param_kernel(Blob<BYTES> p, int* out) {
  if (threadIdx.x == 0 && p.b[BYTES - 1] == 123) out[0] = 1;
}
#include <chrono>
extern "C" double mb_launch_us(int bytes, int reps, void* st) {
  int* out = nullptr;
  cudaMalloc(&out, 64);
  auto run = [&](auto blob) {
    auto t0 = std::chrono::high_resolution_clock::now();
    for (int i = 0; i < reps; ++i) param_kernel<<<1, 32, 0, (cudaStream_t)st>>>(blob, out);
    auto t1 = std::chrono::high_resolution_clock::now();
    cudaStreamSynchronize((cudaStream_t)st);
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
  };
  double r = -1;
  if (bytes == 256) { Blob<256> b{}; run(b); r = run(b); }
  if (bytes == 4096) { Blob<4096> b{}; run(b); r = run(b); }
  if (bytes == 16384) { Blob<16384> b{}; run(b); r = run(b); }
  if (bytes == 30000) { Blob<30000> b{}; run(b); r = run(b); }
  cudaFree(out);
  return r;
}
