// Single rank-1 lattice path (Algorithm 5 of the reference engine,
// lattice_kind = "single"): component-by-component search, residue scatter
// for lattice evaluation.  Reference: construct.py:212-278 (CBC),
// transform.py:67-96 (eval_on_lattice, invert_single).
//
// CBC step t, size M: the smallest z_t in [0, M) for which
//   r_i(z) = (prefix_res_i + col_i * z) mod M
// are pairwise distinct over the distinct (t+1)-prefixes i.  A batch of Z
// candidate values is tested at once: thread (i, z) sets bit r_i(z) in z's
// bitmap with atomicOr and flags z when the bit was already set.
#include "common.cuh"
#include "plan.cuh"

namespace sfft {

__global__ void cbc_scan_kernel(const int64_t* __restrict__ prefix_res, const int32_t* __restrict__ col,
                                int64_t n, int64_t m, int64_t z0, int Z, uint32_t* __restrict__ bits,
                                int64_t words, int32_t* __restrict__ dup) {
  const int zi = blockIdx.y;
  const int64_t z = z0 + zi;
  uint32_t* bm = bits + (int64_t)zi * words;
  const uint64_t mm = (uint64_t)m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = col[i] % m;
    if (c < 0) c += m;
    const uint64_t r = ((uint64_t)prefix_res[i] + ((uint64_t)c * (uint64_t)z) % mm) % mm;
    const uint32_t bit = 1u << (r & 31);
    const uint32_t old = atomicOr(&bm[r >> 5], bit);
    if (old & bit) dup[zi] = 1;
  }
}

int launch_cbc_scan(const int64_t* prefix_res, const int32_t* col, int64_t n, int64_t m, int64_t z0,
                    int Z, uint32_t* bits, int64_t words, int32_t* dup, int num_sms, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(bits, 0, (size_t)Z * words * sizeof(uint32_t), st);
  if (e != cudaSuccess) return (int)e;
  e = cudaMemsetAsync(dup, 0, (size_t)Z * sizeof(int32_t), st);
  if (e != cudaSuccess) return (int)e;
  if (n == 0 || Z == 0) return 0;
  int bx = (int)((n + 255) / 256);
  const int cap = (num_sms * 16 + Z - 1) / Z + 1;
  if (bx > cap) bx = cap;
  cbc_scan_kernel<<<dim3(bx, Z), 256, 0, st>>>(prefix_res, col, n, m, z0, Z, bits, words, dup);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// flag[i] = 1 if row i of a lexicographically sorted set starts a new
// (t1)-prefix (np.unique of the projection onto the first t1 components)
__global__ void prefix_flags_kernel(const int32_t* __restrict__ freqs, int64_t n, int t1,
                                    uint8_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint8_t f = (i == 0);
    if (!f)
      for (int c = 0; c < t1; ++c)
        if (freqs[(int64_t)c * n + i] != freqs[(int64_t)c * n + i - 1]) { f = 1; break; }
    flags[i] = f;
  }
}

int launch_prefix_flags(const int32_t* freqs, int64_t n, int t1, uint8_t* flags, int num_sms,
                        cudaStream_t st) {
  if (n == 0) return 0;
  int64_t want = (n + 255) / 256, cap = (int64_t)num_sms * 8;
  prefix_flags_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(freqs, n, t1, flags);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// acc[k . z mod M] += coef (eval_on_lattice's np.add.at, transform.py:75-78).
// Collisions are summed with atomics (order-dependent only when the lattice
// is not reconstructing for the spectrum).
template <bool FAST>
__global__ void scatter_residues_kernel(const int32_t* __restrict__ freqs, int64_t n, LatTable lt,
                                        const double2* __restrict__ coef, double2* __restrict__ acc) {
  const int d = lt.d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t k[SFFT_DMAX];
    for (int c = 0; c < d; ++c) k[c] = freqs[(int64_t)c * n + i];
    int64_t acc_r = 0;
    const int64_t m = lt.m[0];
    for (int c = 0; c < d; ++c) {
      const int64_t km = mod_slow((int64_t)k[c], m);
      acc_r = (acc_r + (int64_t)(((uint64_t)km * (uint64_t)lt.z[c]) % (uint64_t)m)) % m;
    }
    const double2 v = coef[i];
    atomicAdd(&acc[acc_r].x, v.x);
    atomicAdd(&acc[acc_r].y, v.y);
  }
}

int launch_scatter_residues(const int32_t* freqs, int64_t n, const LatTable& lt, const double2* coef,
                            double2* acc, int num_sms, cudaStream_t st) {
  if (n == 0) return 0;
  int64_t want = (n + 255) / 256, cap = (int64_t)num_sms * 8;
  scatter_residues_kernel<false><<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(freqs, n, lt, coef, acc);
  SFFT_CHECK_LAUNCH();
  return 0;
}

}  // namespace sfft
