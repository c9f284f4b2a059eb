// Shared device helpers for the MR1L hot path (sm_100a).
//
// Exact residue arithmetic: every lattice size M satisfies 1 <= M <= 2^31-1
// (reference lattice.py:36-38, 290-294), so a single product of two residues
// fits in 62 bits.  The fast reduction below needs |x| < 2^52, which the host
// checks before it selects the FAST template variants; the slow variants use
// 64-bit integer division and are exact for every admissible input.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <unordered_map>

#define SFFT_DMAX 64          // largest dimension handled by the device kernels
#define SFFT_LMAX 64          // masks are one uint64 word per candidate

namespace sfft {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a kernel needs
// more than it was already granted on this device (the attribute persists;
// setting it on every launch cost microseconds of host time per call).
inline cudaError_t set_smem_once(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> granted[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = granted[dev].find(fn);
    if (it != granted[dev].end() && it->second >= (int)bytes) return cudaSuccess;
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> g(mu);
    int& v = granted[dev][fn];
    if ((int)bytes > v) v = (int)bytes;
  }
  return e;
}

// number of kernels this library has launched (reported by sfft_launch_count)
inline std::atomic<long long> g_launches{0};

// Optional CUDA-event brackets around kernel classes (sfft_profile_enable):
// the bench reads each class's device time on the launching stream.
enum ProfClass { PROF_SAMPLE = 0, PROF_FFT = 1, PROF_ALIAS = 2, PROF_GATHER = 3, PROF_NCLASS = 4 };
void prof_mark(int cls, bool begin, cudaStream_t st);  // no-op unless enabled

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// x mod m in [0, m) for |x| < 2^52 and 1 <= m < 2^31 (inv_m = 1.0 / m).
// Bluestein chirp c_n = e^{-pi i (n^2 mod 2M) / M} (0 <= n < M < 2^31), the
// value lattice_tables_kernel stores: n^2 mod 2M exactly by a Barrett step
// (inv2m = floor((2^64 - 1) / 2M): the estimate is at most 2 below the
// quotient), then the same sincospi call, so table and recomputation agree
// bit for bit.
__device__ __forceinline__ double2 chirp_at(int64_t n, int64_t m, uint64_t inv2m) {
  const uint64_t m2 = 2 * (uint64_t)m;
  const uint64_t x = (uint64_t)n * (uint64_t)n;
  uint64_t r = x - __umul64hi(x, inv2m) * m2;
  if (r >= m2) r -= m2;
  if (r >= m2) r -= m2;
  double s, c;
  sincospi((double)r / (double)m, &s, &c);
  return make_double2(c, -s);
}

__device__ __forceinline__ int64_t mod_fast(int64_t x, int64_t m, double inv_m) {
  int64_t q = (int64_t)floor((double)x * inv_m);
  int64_t r = x - q * m;
  if (r < 0) r += m;
  else if (r >= m) r -= m;
  return r;
}

// x mod m in [0, m) for any int64 x.
__device__ __forceinline__ int64_t mod_slow(int64_t x, int64_t m) {
  int64_t r = x % m;
  return r < 0 ? r + m : r;
}

// (a * b) mod m for 0 <= a, b < m < 2^31.
template <bool FAST>
__device__ __forceinline__ int64_t mulmod(int64_t a, int64_t b, int64_t m, double inv_m) {
  if (FAST) return mod_fast(a * b, m, inv_m);
  return (int64_t)(((uint64_t)a * (uint64_t)b) % (uint64_t)m);
}

// Components of candidate i of a component-major (d x n) int32 set into
// registers: one pointer walk (a 64-bit add per component) instead of a
// 64-bit multiply-add address per component.
template <int DM>
__device__ __forceinline__ void load_cand(int32_t (&k)[DM], const int32_t* __restrict__ freqs, int64_t n,
                                          int64_t i, int d, bool live = true) {
  const int32_t* p = freqs + i;
#pragma unroll
  for (int c = 0; c < DM; ++c) {
    k[c] = (live && c < d) ? __ldg(p) : 0;
    p += n;
  }
}

// Residue k . z mod M of one candidate (components in registers).
// FAST requires sum_c |k_c| * z_c < 2^52 (host-checked); with i32 != 0 the
// host has also checked d * kmax * M < 2^31, and the sum runs in int32 plus a
// 32-bit Barrett reduction of acc + off32 (off32 = M * d * kmax, a multiple of
// M making the argument non-negative and < 2^32; mu32 = floor((2^32-1)/M),
// quotient low by at most one).  Matches reference lattice.py:511-517
// (componentwise-reduced inner product) exactly in every mode.
template <int DM, bool FAST>
__device__ __forceinline__ int64_t residue(const int32_t (&k)[DM], int d, const int32_t* z,
                                           int64_t m, double inv_m, int i32 = 0,
                                           uint32_t off32 = 0, uint32_t mu32 = 0) {
  if (FAST && i32) {
    int32_t acc = 0;
#pragma unroll
    for (int c = 0; c < DM; ++c)
      if (c < d) acc += k[c] * z[c];
    const uint32_t x = (uint32_t)acc + off32;
    const uint32_t mm = (uint32_t)m;
    uint32_t r = x - __umulhi(x, mu32) * mm;
    if (r >= mm) r -= mm;
    return (int64_t)r;
  }
  if (FAST) {
    int64_t acc = 0;
#pragma unroll
    for (int c = 0; c < DM; ++c)
      if (c < d) acc += (int64_t)k[c] * (int64_t)z[c];
    return mod_fast(acc, m, inv_m);
  } else {
    int64_t acc = 0;
#pragma unroll
    for (int c = 0; c < DM; ++c)
      if (c < d) {
        int64_t km = mod_slow((int64_t)k[c], m);
        acc = (acc + (int64_t)(((uint64_t)km * (uint64_t)z[c]) % (uint64_t)m)) % m;
      }
    return acc;
  }
}

// Block-wide inclusive sum over 32-bit values (blockDim.x multiple of 32, <= 1024).
__device__ __forceinline__ int block_sum(int v, int* smem32) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) smem32[wid] = v;
  __syncthreads();
  int tot = 0;
  if (threadIdx.x < 32) {
    int x = (threadIdx.x < (blockDim.x >> 5)) ? smem32[threadIdx.x] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    tot = x;
  }
  return tot;  // valid in thread 0
}

}  // namespace sfft

// every kernel launch is followed by SFFT_CHECK_LAUNCH() (one launch) or
// SFFT_CHECK_LAUNCHES(n) (n launches since the last check)
#define SFFT_CHECK_LAUNCHES(n)                        \
  do {                                                \
    ::sfft::g_launches += (n);                        \
    cudaError_t _e = cudaGetLastError();              \
    if (_e != cudaSuccess) return (int)_e;            \
  } while (0)
#define SFFT_CHECK_LAUNCH() SFFT_CHECK_LAUNCHES(1)
