// K2: batched prime-length DFT by Bluestein's algorithm on power-of-two
// four-step Stockham FFTs (replaces reference transform.py:50-64, the
// scipy.fft.fft call at transform.py:61, used by invert_multiple :121).
//
// For a lattice of prime size M, with chirp c_n = e^{-pi i (n^2 mod 2M) / M}:
//     X_k = c_k * sum_n (x_n c_n) * conj(c_{k-n})            (k < M)
// i.e. a linear convolution evaluated as a cyclic one of length
// P = 2^p >= 2M - 1.  The chirp exponent is reduced mod 2M in integers so
// the phase is exact for every M < 2^31 (SURVEY §7 hard part 3).
//
// Layout of one transform buffer (P complex128): natural index n.  The FFT
// of length P = P1 * P2 (P2 = 2^min(11,p), 4096 for p > 22) runs as
//   column pass  : P2 columns of length P1 (stride P2) + twiddle e^{-2pi i n2 k1/P}
//   row pass     : P1 rows of length P2, fused: forward FFT, * Bhat, inverse
//                  FFT, * e^{+2pi i n2 k1 / P}
//   column pass  : inverse length-P1 FFTs, then the post-chirp, written only
//                  for n < M.
// Bhat = FFT_P(b) / P with b_m = conj(c_m) wrapped cyclically is built once per
// lattice by the same forward passes (row pass in FWD_ONLY mode), so its
// layout matches the data after the forward row FFT by construction.
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

#include <cstdlib>
#include "fft.cuh"
#include "plan.cuh"

namespace sfft {

// ---------------------------------------------------------------------------
// tables

// twiddle/chirp tables: tw[n] = e^{+2pi i n/M}, chirp[n] = e^{-pi i (n^2 mod 2M)/M}
__global__ void lattice_tables_kernel(LatTable lt, double2* __restrict__ tw,
                                      double2* __restrict__ chirp) {
  const int l = blockIdx.y;
  const int64_t m = lt.m[l];
  const int64_t off = lt.off[l];
  const uint64_t inv2m = ~0ull / (2 * (uint64_t)m);
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < m;
       n += (int64_t)gridDim.x * blockDim.x) {
    double s, c;
    // e^{+2 pi i n / M}: argument 2n/M for sincospi
    sincospi(2.0 * (double)n / (double)m, &s, &c);
    tw[off + n] = make_double2(c, s);
    chirp[off + n] = chirp_at(n, m, inv2m);
  }
}

// FFT tables for one P: [twP1 | twP2 | Tlo | Thi], all e^{-2 pi i m / N}
__global__ void fft_tables_kernel(FftGeom g, double2* __restrict__ out) {
  const int64_t total = g.table_len;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    double num, den;
    if (i < g.P1) { num = (double)i; den = (double)g.P1; }
    else if (i < g.P1 + g.P2) { num = (double)(i - g.P1); den = (double)g.P2; }
    else if (i < g.P1 + g.P2 + g.nlo) { num = (double)(i - g.P1 - g.P2); den = (double)g.P; }
    else { num = (double)((i - g.P1 - g.P2 - g.nlo) << g.qlo); den = (double)g.P; }
    double s, c;
    sincospi(2.0 * num / den, &s, &c);
    out[i] = make_double2(c, -s);
  }
}

// Bluestein kernel sequence b: b[m] = e^{+pi i (m^2 mod 2M)/M} for m < M,
// b[P-m] = b[m] for 0 < m < M, zero elsewhere.  One row of `bhat` per lattice.
__global__ void bluestein_b_kernel(LatTable lt, const double2* __restrict__ chirp,
                                   double2* __restrict__ bhat, int64_t P) {
  const int l = blockIdx.y;
  const int64_t m = lt.m[l];
  const double2* ch = chirp + lt.off[l];
  double2* b = bhat + (int64_t)l * P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (i < m) v = cconj(ch[i]);
    else if (P - i < m) v = cconj(ch[P - i]);
    b[i] = v;
  }
}

// ---------------------------------------------------------------------------
// column pass (P1 = 2^LOG1 > 1, P2 = TE).  CTA = C = TE/P1 consecutive
// columns of one unit.  FWD: mask n >= M to zero if mask_input, forward FFT,
// twiddle, store transposed.  INV: inverse FFT, post-chirp, store n < M.
template <int LOG1, bool INV, int TE>
__global__ void __launch_bounds__(FFT_T, TE == 2048 ? 4 : 2)
fft_col_kernel(double2* __restrict__ buf, int64_t ustride, UnitTable ut, FftGeom g, int mask_input,
               const double2* __restrict__ ftab, const double2* __restrict__ chirp) {
  extern __shared__ double2 s[];
  constexpr int P1 = 1 << LOG1;
  constexpr int P2 = TE;  // the row length equals the tile size
  constexpr int C = TE / P1;
  constexpr int rstride = Tile<TE>::rstride(P1);
  const int u = blockIdx.y;
  const int c0 = blockIdx.x * C;
  const int lat = ut.lat[u];
  const int64_t m = ut.m[lat];
  double2* ub = buf + (int64_t)u * ustride;

  // load (coalesced along columns), transpose into rows of length P1
#pragma unroll
  for (int f = threadIdx.x; f < TE; f += FFT_T) {
    const int c = f % C, n1 = f / C;
    const int64_t n = (int64_t)n1 * P2 + c0 + c;
    double2 v;
    if (!INV && mask_input && n >= m) v = make_double2(0.0, 0.0);
    else v = ub[n];
    s[c * rstride + Tile<TE>::pad(n1)] = v;
  }
  __syncthreads();
  block_fft<LOG1, INV, TE>(s, ftab + g.off_p1);
  if (!INV && C <= FFT_T) {
    // this thread's elements share the column n2 and step k1 by FFT_T / C:
    // twiddles e^{-2 pi i n2 k1 / P} by a short recurrence from two table
    // lookups (the per-element two-level lookups were the LSU's largest
    // global-load consumer)
    const int c = threadIdx.x % C;
    const int64_t n2 = c0 + c;
    double2 w = twP(g, ftab, n2 * (int64_t)(threadIdx.x / C));
    const double2 step = twP(g, ftab, n2 * (int64_t)(FFT_T / C));
#pragma unroll
    for (int f = threadIdx.x; f < TE; f += FFT_T) {
      const int k1 = f / C;
      const double2 v = cmul(s[c * rstride + Tile<TE>::pad(k1)], w);
      ub[(int64_t)k1 * P2 + n2] = v;
      w = cmul(w, step);
    }
  } else if (!INV) {
#pragma unroll
    for (int f = threadIdx.x; f < TE; f += FFT_T) {
      const int c = f % C, k1 = f / C;
      const int64_t n2 = c0 + c;
      double2 v = s[c * rstride + Tile<TE>::pad(k1)];
      v = cmul(v, twP(g, ftab, n2 * (int64_t)k1));
      ub[(int64_t)k1 * P2 + n2] = v;
    }
  } else {
    // post-chirp: all chirp loads first, then multiply + store (one exposed
    // latency instead of one per group of four)
    // (chirp == nullptr: recomputed, not read -- see chirp_at)
    const double2* ch = chirp ? chirp + ut.off[lat] : nullptr;
    const uint64_t inv2m = ~0ull / (2 * (uint64_t)m);
    constexpr int Q = TE / FFT_T;
    double2 cv[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int f = threadIdx.x + q * FFT_T;
      const int64_t n = (int64_t)(f / C) * P2 + c0 + f % C;
      cv[q] = n < m ? (ch ? __ldg(&ch[n]) : chirp_at(n, m, inv2m)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int f = threadIdx.x + q * FFT_T;
      const int c = f % C, n1 = f / C;
      const int64_t n = (int64_t)n1 * P2 + c0 + c;
      if (n < m) ub[n] = cmul(s[c * rstride + Tile<TE>::pad(n1)], cv[q]);
    }
  }
}

// ---------------------------------------------------------------------------
// row pass (P2 = 2^LOG2).  CTA = TE/P2 rows (rows index (unit, k1) flattened).
// MODE 0 (conv): forward FFT, * bhat, inverse FFT, then twiddle (P1 > 1) or
//                post-chirp (P1 == 1, whole transform in one row).
// MODE 1 (fwd only, builds bhat): forward FFT, scale by 1/P.
template <int LOG2, int MODE, int TE>
__global__ void __launch_bounds__(FFT_T, TE == 2048 ? 4 : 2)
fft_row_kernel(double2* __restrict__ buf, int64_t ustride, UnitTable ut, FftGeom g, int total_rows,
               const double2* __restrict__ ftab, const double2* __restrict__ bhat,
               const double2* __restrict__ chirp) {
  extern __shared__ double2 s[];
  constexpr int P2 = 1 << LOG2;
  constexpr int rows = TE / P2;
  constexpr int rstride = Tile<TE>::rstride(P2);
  const int P1 = g.P1;
  const int g0 = blockIdx.x * rows;
  const bool single = (P1 == 1);

  // all loads first, then the shared-memory stores: keeps the 16 loads of a
  // thread in flight together (interleaved, ptxas serialised them)
  constexpr int Q = TE / FFT_T;
  double2 v[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int f = threadIdx.x + q * FFT_T;
    const int r = f / P2, i = f % P2;
    const int grow = g0 + r;
    v[q] = make_double2(0.0, 0.0);
    if (grow < total_rows) {
      const int u = grow / P1, k1 = grow - u * P1;
      const int lat = ut.lat[u];
      if (!(MODE == 0 && single && i >= ut.m[lat]))
        v[q] = __ldcs(&buf[(int64_t)u * ustride + (int64_t)k1 * P2 + i]);
    }
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int f = threadIdx.x + q * FFT_T;
    s[(f / P2) * rstride + Tile<TE>::pad(f % P2)] = v[q];
  }
  __syncthreads();
  block_fft<LOG2, false, TE>(s, ftab + g.off_p2);
  if (MODE == 1) {
    const double scale = 1.0 / (double)g.P;  // exact when P is a power of two
#pragma unroll
    for (int f = threadIdx.x; f < TE; f += FFT_T) {
      const int r = f / P2, i = f % P2;
      const int grow = g0 + r;
      if (grow < total_rows) {
        const int u = grow / P1, k1 = grow - u * P1;
        double2 v = s[r * rstride + Tile<TE>::pad(i)];
        buf[(int64_t)u * ustride + (int64_t)k1 * P2 + i] = make_double2(v.x * scale, v.y * scale);
      }
    }
    return;
  }
  // pointwise product with Bhat (same layout); loads first (see above)
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int f = threadIdx.x + q * FFT_T;
    const int r = f / P2, i = f % P2;
    const int grow = g0 + r;
    v[q] = make_double2(0.0, 0.0);
    if (grow < total_rows) {
      const int u = grow / P1, k1 = grow - u * P1;
      v[q] = __ldg(&bhat[(int64_t)ut.lat[u] * ustride + (int64_t)k1 * P2 + i]);
    }
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int f = threadIdx.x + q * FFT_T;
    const int si = (f / P2) * rstride + Tile<TE>::pad(f % P2);
    s[si] = cmul(s[si], v[q]);
  }
  __syncthreads();
  block_fft<LOG2, true, TE>(s, ftab + g.off_p2);
  if (rows == 1 && !single) {
    // one row k1 per CTA: e^{+2 pi i i k1 / P} for i = tid + FFT_T q by a short
    // recurrence from two table lookups (see the column pass)
    if (g0 >= total_rows) return;
    const int u = g0 / P1, k1 = g0 - u * P1;
    double2* ub = buf + (int64_t)u * ustride + (int64_t)k1 * P2;
    double2 w = twP(g, ftab, (int64_t)threadIdx.x * k1);
    const double2 step = twP(g, ftab, (int64_t)FFT_T * k1);
#pragma unroll
    for (int i = threadIdx.x; i < P2; i += FFT_T) {
      ub[i] = cmulc(s[Tile<TE>::pad(i)], w);
      w = cmul(w, step);
    }
    return;
  }
#pragma unroll
  for (int f = threadIdx.x; f < TE; f += FFT_T) {
    const int r = f / P2, i = f % P2;
    const int grow = g0 + r;
    if (grow < total_rows) {
      const int u = grow / P1, k1 = grow - u * P1;
      const int lat = ut.lat[u];
      double2 v = s[r * rstride + Tile<TE>::pad(i)];
      double2* ub = buf + (int64_t)u * ustride;
      if (!single) {
        v = cmulc(v, twP(g, ftab, (int64_t)i * k1));  // e^{+2 pi i n2 k1 / P}
        ub[(int64_t)k1 * P2 + i] = v;
      } else if (i < ut.m[lat]) {
        ub[i] = cmul(v, __ldg(&chirp[ut.off[lat] + i]));
      }
    }
  }
}

// Row pass specialised for rows of P2 = 2048 in 2048-element tiles (one row
// per CTA, thread t holds elements t + 256 q, q < 8): the radix-8 first pass
// of each FFT reads the thread's registers (the coalesced row load, or the
// pointwise product), and the radix-4 last pass leaves its outputs in the
// same registers (element j + 512 r of butterfly j = t + 256 q is slot
// q + 2 r), so the Bhat product and the final store need no shared-memory
// round trip: 6 instead of 10 shared-memory passes per row, same arithmetic
// (bit-identical to fft_row_kernel).
template <bool INV>
__device__ __forceinline__ void row2048_first_pass(double2 (&v)[8], double2* s) {
  dft_reg<8, INV>(v);
#pragma unroll
  for (int r = 0; r < 8; ++r) s[Tile<2048>::pad(threadIdx.x * 8 + r)] = v[bitrev_small(r, 3)];
  __syncthreads();
}

template <bool INV>
__device__ __forceinline__ void row2048_last_pass(double2 (&v)[8], const double2* s,
                                                  const double2* __restrict__ twN) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = threadIdx.x + q * FFT_T;
    double2 w[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) w[r] = s[Tile<2048>::pad(j + r * 512)];
    twiddle_reg<4, INV>(w, j, 1, twN);
    dft_reg<4, INV>(w);
#pragma unroll
    for (int r = 0; r < 4; ++r) v[q + 2 * r] = w[bitrev_small(r, 2)];
  }
}

template <int MODE>
__global__ void __launch_bounds__(FFT_T, MODE == 0 ? 3 : 4)  // MODE 0: + 32 KB Bhat staging -> 3 CTAs/SM
fft_row2048_kernel(double2* __restrict__ buf, int64_t ustride, UnitTable ut, FftGeom g, int total_rows,
                   const double2* __restrict__ ftab, const double2* __restrict__ bhat) {
  extern __shared__ double2 s[];
  constexpr int N = 2048;
  constexpr int rstride = Tile<2048>::rstride(N);
  const int grow = blockIdx.x;
  if (grow >= total_rows) return;
  // k1 outer, unit inner: the rows of all units at one k1 run in neighbouring
  // CTAs, so the units that share a lattice (the r~ iterations of a step)
  // read its Bhat row from L2 -- one HBM read per lattice instead of per unit
  const int nu = ut.nunits;
  const int k1 = grow / nu, u = grow - k1 * nu;
  double2* row = buf + (int64_t)u * ustride + (int64_t)k1 * N;
  const double2* twN = ftab + g.off_p2;
  double2* bsm = s + rstride;  // MODE 0: the Bhat row, prefetched into shared memory (cp.async)
  if (MODE == 0) {
    const double2* bh = bhat + (int64_t)ut.lat[u] * ustride + (int64_t)k1 * N;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&bsm[threadIdx.x + q * FFT_T]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(&bh[threadIdx.x + q * FFT_T])
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  double2 v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = __ldcs(&row[threadIdx.x + q * FFT_T]);
  row2048_first_pass<false>(v, s);
  stockham_pass<8, false, 2048>(s, 1, rstride, N, 8, twN);
  stockham_pass<8, false, 2048>(s, 1, rstride, N, 64, twN);
  row2048_last_pass<false>(v, s, twN);
  if (MODE == 1) {
    const double scale = 1.0 / (double)g.P;
#pragma unroll
    for (int q = 0; q < 8; ++q) row[threadIdx.x + q * FFT_T] = make_double2(v[q].x * scale, v[q].y * scale);
    return;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");  // each thread reads back its own copies only
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = cmul(v[q], bsm[threadIdx.x + q * FFT_T]);
  __syncthreads();  // every thread's last-pass reads are done before the smem is rewritten
  row2048_first_pass<true>(v, s);
  stockham_pass<8, true, 2048>(s, 1, rstride, N, 8, twN);
  stockham_pass<8, true, 2048>(s, 1, rstride, N, 64, twN);
  row2048_last_pass<true>(v, s, twN);
  // e^{+2 pi i i k1 / P} for i = t + 256 q by a short recurrence (see the column pass)
  double2 w = twP(g, ftab, (int64_t)threadIdx.x * k1);
  const double2 step = twP(g, ftab, (int64_t)FFT_T * k1);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    row[threadIdx.x + q * FFT_T] = cmulc(v[q], w);
    w = cmul(w, step);
  }
}

template <int MODE>
static int launch_row2048(unsigned blocks, cudaStream_t st, double2* buf, int64_t us, const UnitTable& ut,
                          const FftGeom& g, int total_rows, const double2* ftab, const double2* bhat) {
  const size_t sm = ((size_t)Tile<2048>::rstride(2048) + (MODE == 0 ? 2048 : 0)) * sizeof(double2);
  cudaError_t e = set_smem_once((const void*)fft_row2048_kernel<MODE>, sm);
  if (e != cudaSuccess) return (int)e;
  fft_row2048_kernel<MODE><<<blocks, FFT_T, sm, st>>>(buf, us, ut, g, total_rows, ftab, bhat);
  SFFT_CHECK_LAUNCH();
  return 0;
}

static bool colx2_pow2_enabled() {
  static const bool v = [] {
    const char* e = getenv("SFFT_B200_FFT_COLX2");
    return !(e && strcmp(e, "0") == 0);
  }();
  return v;
}

static bool row2048_enabled() {
  static const bool v = [] {
    const char* e = getenv("SFFT_B200_FFT_ROW2048");
    return !(e && strcmp(e, "0") == 0);
  }();
  return v;
}

// compile-time size dispatch: TE = 2048 for log sizes <= 11, 4096 for 12
// (the column length P1 = 2^11..2^12 of p = 23, 24 also uses 4096 tiles)
template <bool INV>
static int launch_col(int te, int lg, dim3 grid, size_t sm, cudaStream_t st, double2* buf, int64_t us,
                      const UnitTable& ut, const FftGeom& p, int mask, const double2* ftab, const double2* chirp) {
#define SFFT_COL(TEV, L)                                                                         \
  case L: {                                                                                      \
    cudaError_t e = set_smem_once((const void*)fft_col_kernel<L, INV, TEV>, sm);                 \
    if (e != cudaSuccess) return (int)e;                                                         \
    fft_col_kernel<L, INV, TEV><<<grid, FFT_T, sm, st>>>(buf, us, ut, p, mask, ftab, chirp);     \
    break;                                                                                       \
  }
  if (te == 2048) {
    switch (lg) {
      SFFT_COL(2048, 1) SFFT_COL(2048, 2) SFFT_COL(2048, 3) SFFT_COL(2048, 4) SFFT_COL(2048, 5)
      SFFT_COL(2048, 6) SFFT_COL(2048, 7) SFFT_COL(2048, 8) SFFT_COL(2048, 9) SFFT_COL(2048, 10)
      SFFT_COL(2048, 11)
      default: return -22;
    }
  } else {
    switch (lg) {
      SFFT_COL(4096, 11) SFFT_COL(4096, 12)
      default: return -22;
    }
  }
#undef SFFT_COL
  SFFT_CHECK_LAUNCH();
  return 0;
}

template <int MODE>
static int launch_row(int te, int lg, unsigned blocks, size_t sm, cudaStream_t st, double2* buf, int64_t us,
                      const UnitTable& ut, const FftGeom& p, int total_rows, const double2* ftab,
                      const double2* bhat, const double2* chirp) {
#define SFFT_ROW(TEV, L)                                                                         \
  case L: {                                                                                      \
    cudaError_t e = set_smem_once((const void*)fft_row_kernel<L, MODE, TEV>, sm);                \
    if (e != cudaSuccess) return (int)e;                                                         \
    fft_row_kernel<L, MODE, TEV><<<blocks, FFT_T, sm, st>>>(buf, us, ut, p, total_rows, ftab, bhat, \
                                                            chirp);                              \
    break;                                                                                       \
  }
  if (te == 2048) {
    switch (lg) {
      SFFT_ROW(2048, 4) SFFT_ROW(2048, 5) SFFT_ROW(2048, 6) SFFT_ROW(2048, 7) SFFT_ROW(2048, 8)
      SFFT_ROW(2048, 9) SFFT_ROW(2048, 10) SFFT_ROW(2048, 11)
      default: return -22;
    }
  } else {
    switch (lg) {
      SFFT_ROW(4096, 12)
      default: return -22;
    }
  }
#undef SFFT_ROW
  SFFT_CHECK_LAUNCH();
  return 0;
}

static size_t fft_smem_bytes(int te, int rows_len) {
  const int rows = te / rows_len;
  const int rs = te == 2048 ? Tile<2048>::rstride(rows_len) : Tile<4096>::rstride(rows_len);
  return (size_t)rows * rs * sizeof(double2);
}

int launch_fft_tables(const FftGeom& g, double2* out, cudaStream_t st) {
  int blocks = (int)((g.table_len + 255) / 256);
  if (blocks > 1024) blocks = 1024;
  fft_tables_kernel<<<blocks, 256, 0, st>>>(g, out);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_lattice_tables(const LatTable& lt, double2* tw, double2* chirp, cudaStream_t st) {
  int64_t mmax = 1;
  for (int l = 0; l < lt.nlat; ++l) mmax = lt.m[l] > mmax ? lt.m[l] : mmax;
  int bx = (int)((mmax + 255) / 256);
  if (bx > 512) bx = 512;
  lattice_tables_kernel<<<dim3(bx, lt.nlat), 256, 0, st>>>(lt, tw, chirp);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// forward passes on `nunits` buffers (column pass if P1 > 1, then row pass in `mode`)
static int run_cols(bool inv, double2* buf, int64_t ustride, const UnitTable& ut, const FftGeom& g, int mask,
                    const double2* ftab, const double2* chirp, cudaStream_t st) {
  if (g.P1 == 1) return 0;
  dim3 grid(g.P2 / fft_col_ctas_cols(g.P1, g.te), ut.nunits);
  if (g.f1 > 1 || (g.te == 2048 && g.a1 >= 4 && colx2_pow2_enabled()))
    return launch_colx(inv, g, grid, st, buf, ustride, ut, mask, ftab, chirp);
  const size_t sm = fft_smem_bytes(g.te, g.P1);
  return inv ? launch_col<true>(g.te, g.a1, grid, sm, st, buf, ustride, ut, g, mask, ftab, chirp)
             : launch_col<false>(g.te, g.a1, grid, sm, st, buf, ustride, ut, g, mask, ftab, chirp);
}

int launch_bhat(const LatTable& lt, const double2* chirp, double2* bhat, const FftGeom& g,
                const double2* ftab, cudaStream_t st) {
  const int64_t P = g.P;
  int bx = (int)((P + 255) / 256);
  if (bx > 512) bx = 512;
  bluestein_b_kernel<<<dim3(bx, lt.nlat), 256, 0, st>>>(lt, chirp, bhat, P);
  SFFT_CHECK_LAUNCH();
  UnitTable ut;
  ut.nunits = lt.nlat;
  ut.nlat = lt.nlat;
  for (int l = 0; l < lt.nlat; ++l) { ut.lat[l] = l; ut.m[l] = lt.m[l]; ut.off[l] = lt.off[l]; }
  int rc = run_cols(false, bhat, P, ut, g, 0, ftab, chirp, st);
  if (rc) return rc;
  const size_t sm = fft_smem_bytes(g.te, g.P2);
  const int total_rows = ut.nunits * g.P1;
  const int rows = g.te / g.P2;
  if (g.te == 2048 && g.P2 == 2048 && g.P1 > 1 && row2048_enabled())
    return launch_row2048<1>(total_rows, st, bhat, P, ut, g, total_rows, ftab, nullptr);
  return launch_row<1>(g.te, g.p2, (total_rows + rows - 1) / rows, sm, st, bhat, P, ut, g, total_rows,
                       ftab, nullptr, chirp);
}

// drop the dead tail [M, P) of a unit's buffer from L2 without writing it
// back (discard.global.L2): after the inverse column pass only the spectrum
// k < M is live, the tail holds row-pass data nobody reads again
__global__ void discard_tails_kernel(double2* __restrict__ buf, int64_t ustride, UnitTable ut, int64_t P) {
  const int u = blockIdx.y;
  const int64_t M = ut.m[ut.lat[u]];
  const uintptr_t base = (uintptr_t)(buf + (int64_t)u * ustride);
  const uintptr_t a = (base + (uintptr_t)M * sizeof(double2) + 127) & ~(uintptr_t)127;
  const uintptr_t e = (base + (uintptr_t)P * sizeof(double2)) & ~(uintptr_t)127;
  for (uintptr_t p = a + ((uintptr_t)blockIdx.x * blockDim.x + threadIdx.x) * 128; p < e;
       p += (uintptr_t)gridDim.x * blockDim.x * 128)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// The inverse column pass recomputes the post-chirp (chirp_at, bit-identical
// to the table) instead of reading 16 B per output point from the lattice
// table; SFFT_B200_CHIRP_TABLE=1 reads the table (A/B).
static bool post_chirp_table() {
  static const bool v = [] {
    const char* e = getenv("SFFT_B200_CHIRP_TABLE");
    return e && strcmp(e, "1") == 0;
  }();
  return v;
}

static int bluestein_group(double2* buf, const UnitTable& ut, const FftGeom& g, const double2* ftab,
                           const double2* bhat, const double2* chirp, bool discard, cudaStream_t st) {
  const int64_t P = g.P;
  int rc = run_cols(false, buf, P, ut, g, 1, ftab, chirp, st);
  if (rc) return rc;
  const size_t sm = fft_smem_bytes(g.te, g.P2);
  const int total_rows = ut.nunits * g.P1;
  const int rows = g.te / g.P2;
  if (g.te == 2048 && g.P2 == 2048 && g.P1 > 1 && row2048_enabled())
    rc = launch_row2048<0>(total_rows, st, buf, P, ut, g, total_rows, ftab, bhat);
  else
    rc = launch_row<0>(g.te, g.p2, (total_rows + rows - 1) / rows, sm, st, buf, P, ut, g, total_rows, ftab,
                       bhat, chirp);
  if (rc) return rc;
  rc = run_cols(true, buf, P, ut, g, 0, ftab, post_chirp_table() ? chirp : nullptr, st);
  if (rc || !discard) return rc;
  discard_tails_kernel<<<dim3(64, ut.nunits), 256, 0, st>>>(buf, P, ut, P);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// SFFT_B200_FFT_GROUP_MB=<MB> runs the three passes on groups of units whose
// P-length buffers fit in L2 together (the column pass's output read back by
// the row pass from L2, dead tails discarded).  Off by default: at config 1
// it cut DRAM traffic but the smaller launches' tails cost more than the
// traffic saved (K2 0.184 -> 0.225 ms with 40 MB groups, profiles/r02_*).
int launch_bluestein(double2* buf, const UnitTable& ut, const FftGeom& g, const double2* ftab,
                     const double2* bhat, const double2* chirp, cudaStream_t st) {
  const int64_t P = g.P;
  static const int64_t budget = [] {
    const char* e = getenv("SFFT_B200_FFT_GROUP_MB");
    return (int64_t)(e ? atof(e) : 0.0) << 20;
  }();
  const int64_t unit_bytes = P * (int64_t)sizeof(double2);
  int per = budget > 0 ? (int)(budget / unit_bytes) : ut.nunits;
  if (per < 1) per = 1;
  const bool grouped = per < ut.nunits && P >= (1 << 18);
  prof_mark(PROF_FFT, true, st);
  int rc = 0;
  if (!grouped) {
    rc = bluestein_group(buf, ut, g, ftab, bhat, chirp, false, st);
  } else {
    UnitTable* sub = new UnitTable(ut);
    for (int u0 = 0; u0 < ut.nunits && !rc; u0 += per) {
      const int nu = ut.nunits - u0 < per ? ut.nunits - u0 : per;
      sub->nunits = nu;
      for (int j = 0; j < nu; ++j) {
        sub->lat[j] = ut.lat[u0 + j];
        sub->it[j] = ut.it[u0 + j];
      }
      rc = bluestein_group(buf + (int64_t)u0 * P, *sub, g, ftab, bhat, chirp, true, st);
    }
    delete sub;
  }
  prof_mark(PROF_FFT, false, st);
  return rc;
}

}  // namespace sfft
