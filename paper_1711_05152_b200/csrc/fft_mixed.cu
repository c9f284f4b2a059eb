// K2 column passes for mixed-radix Bluestein sizes P = P1 * 2048 with
// P1 = f * 2^a, f in {3, 5, 7, 9, 25} (see plan.cuh fft_geom): the same
// passes as fft_col_kernel (fft.cu) over C = 2^c columns of length P1 per
// CTA (C * P1 <= 2048 elements), with the odd radices applied first.
//
// Choosing P among these sizes instead of powers of two cuts the padded
// length from up to 2x (mean 1.43x) of 2M - 1 to at most 1.33x (mean 1.08x):
// every Bluestein pass moves and transforms P points, so K2's time and
// traffic shrink with it (config 1: P = 524288 -> 409600).
#include "common.cuh"
#include "fft.cuh"
#include "plan.cuh"

namespace sfft {

// FWD: mask n >= M to zero if mask_input, forward FFT of length P1, twiddle
// e^{-2 pi i n2 k1 / P}, store transposed (row k1 of length P2).
// INV: inverse FFT of length P1, post-chirp, store n < M.
template <int A, int F, bool INV>
__global__ void __launch_bounds__(FFT_T, 4)
fft_colx_kernel(double2* __restrict__ buf, int64_t ustride, UnitTable ut, FftGeom g, int mask_input,
                const double2* __restrict__ ftab, const double2* __restrict__ chirp) {
  extern __shared__ double2 s[];
  constexpr int P1 = F << A;
  constexpr int P2 = 2048;
  constexpr int C = fft_col_ctas_cols(P1, 2048);
  constexpr int E = C * P1;
  constexpr int rstride = Tile<2048>::rstride(P1);
  const int u = blockIdx.y;
  const int c0 = blockIdx.x * C;
  const int lat = ut.lat[u];
  const int64_t m = ut.m[lat];
  double2* ub = buf + (int64_t)u * ustride;

  // loads first (all in flight), then the transposing shared-memory stores
  constexpr int Q = (E + FFT_T - 1) / FFT_T;
  double2 v[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int f = threadIdx.x + q * FFT_T;
    v[q] = make_double2(0.0, 0.0);
    if (f < E) {
      const int64_t n = (int64_t)(f / C) * P2 + c0 + f % C;
      if (INV || !mask_input || n < m) v[q] = ub[n];
    }
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int f = threadIdx.x + q * FFT_T;
    if (f < E) s[(f % C) * rstride + Tile<2048>::pad(f / C)] = v[q];
  }
  __syncthreads();
  block_fft_x<F, A, INV, C>(s, ftab + g.off_p1);
  if (!INV) {
    if constexpr (C <= FFT_T) {
      // this thread's elements share the column n2 and step k1 by FFT_T / C
      const int c = threadIdx.x % C;
      const int64_t n2 = c0 + c;
      double2 w = twP(g, ftab, n2 * (int64_t)(threadIdx.x / C));
      const double2 step = twP(g, ftab, n2 * (int64_t)(FFT_T / C));
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int f = threadIdx.x + q * FFT_T;
        if (f < E) {
          const int k1 = f / C;
          ub[(int64_t)k1 * P2 + n2] = cmul(s[c * rstride + Tile<2048>::pad(k1)], w);
        }
        w = cmul(w, step);
      }
    } else {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int f = threadIdx.x + q * FFT_T;
        if (f < E) {
          const int c = f % C, k1 = f / C;
          const int64_t n2 = c0 + c;
          ub[(int64_t)k1 * P2 + n2] = cmul(s[c * rstride + Tile<2048>::pad(k1)], twP(g, ftab, n2 * (int64_t)k1));
        }
      }
    }
  } else {
    const double2* ch = chirp + ut.off[lat];
    double2 cv[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int f = threadIdx.x + q * FFT_T;
      const int64_t n = (int64_t)(f / C) * P2 + c0 + f % C;
      cv[q] = (f < E && n < m) ? __ldg(&ch[n]) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int f = threadIdx.x + q * FFT_T;
      const int c = f % C, n1 = f / C;
      const int64_t n = (int64_t)n1 * P2 + c0 + c;
      if (f < E && n < m) ub[n] = cmul(s[c * rstride + Tile<2048>::pad(n1)], cv[q]);
    }
  }
}

template <int A, int F>
static int launch_colx_t(bool inv, const FftGeom& g, dim3 grid, cudaStream_t st, double2* buf, int64_t us,
                         const UnitTable& ut, int mask, const double2* ftab, const double2* chirp) {
  constexpr int P1 = F << A;
  const size_t sm = (size_t)fft_col_ctas_cols(P1, 2048) * Tile<2048>::rstride(P1) * sizeof(double2);
  const void* fn = inv ? (const void*)fft_colx_kernel<A, F, true> : (const void*)fft_colx_kernel<A, F, false>;
  cudaError_t e = set_smem_once(fn, sm);
  if (e != cudaSuccess) return (int)e;
  if (inv) fft_colx_kernel<A, F, true><<<grid, FFT_T, sm, st>>>(buf, us, ut, g, mask, ftab, chirp);
  else fft_colx_kernel<A, F, false><<<grid, FFT_T, sm, st>>>(buf, us, ut, g, mask, ftab, chirp);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// a = 0 .. amax(F) with F * 2^a <= 2048
template <int F, int A>
static int dispatch_a(int a, bool inv, const FftGeom& g, dim3 grid, cudaStream_t st, double2* buf, int64_t us,
                      const UnitTable& ut, int mask, const double2* ftab, const double2* chirp) {
  if constexpr ((F << A) > 2048) {
    return -22;
  } else {
    if (a == A) return launch_colx_t<A, F>(inv, g, grid, st, buf, us, ut, mask, ftab, chirp);
    return dispatch_a<F, A + 1>(a, inv, g, grid, st, buf, us, ut, mask, ftab, chirp);
  }
}

int launch_colx(bool inv, const FftGeom& g, dim3 grid, cudaStream_t st, double2* buf, int64_t ustride,
                const UnitTable& ut, int mask_input, const double2* ftab, const double2* chirp) {
  if (g.te != 2048 || g.P2 != 2048) return -22;
  switch (g.f1) {
    case 3: return dispatch_a<3, 0>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    case 5: return dispatch_a<5, 0>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    case 7: return dispatch_a<7, 0>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    case 9: return dispatch_a<9, 0>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    case 25: return dispatch_a<25, 0>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    default: return -22;
  }
}

}  // namespace sfft
