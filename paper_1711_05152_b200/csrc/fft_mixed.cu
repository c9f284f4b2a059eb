// K2 column passes for mixed-radix Bluestein sizes P = P1 * 2048 with
// P1 = f * 2^a, f in {3, 5, 7, 9, 25} (see plan.cuh fft_geom): the same
// passes as fft_col_kernel (fft.cu) over C = 2^c columns of length P1 per
// CTA (C * P1 <= 2048 elements), with the odd radices applied first.
//
// Choosing P among these sizes instead of powers of two cuts the padded
// length from up to 2x (mean 1.43x) of 2M - 1 to at most 1.33x (mean 1.08x):
// every Bluestein pass moves and transforms P points, so K2's time and
// traffic shrink with it (config 1: P = 524288 -> 409600).
#include <stdlib.h>
#include <string.h>

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
  constexpr int rstride = rstride_x(P1);
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
    const double2* ch = chirp ? chirp + ut.off[lat] : nullptr;  // nullptr: recomputed (chirp_at)
    const uint64_t inv2m = ~0ull / (2 * (uint64_t)m);
    double2 cv[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int f = threadIdx.x + q * FFT_T;
      const int64_t n = (int64_t)(f / C) * P2 + c0 + f % C;
      cv[q] = (f < E && n < m) ? (ch ? __ldg(&ch[n]) : chirp_at(n, m, inv2m)) : make_double2(0.0, 0.0);
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

// ---------------------------------------------------------------------------
// Register hand-off variant (P1 = f * 2^a with at least two passes): the first
// pass's butterflies read their R0 inputs straight from global memory (lane
// order: column fastest, as the coalesced tile load) and the last pass's
// outputs stay in registers for the twiddle / post-chirp and the store, so
// the transposing shared-memory round trips at both ends are gone (2 instead
// of 4 shared-memory store+load passes for P1 = 200).

// radix of pass i of a column of length F * 2^A: odd radices first (9 = 3.3,
// 25 = 5.5), then radix 8 while >= 3 bits remain, then 4 or 2
template <int F, int A>
struct ColPasses {
  static constexpr int NODD = F == 1 ? 0 : ((F == 9 || F == 25) ? 2 : 1);
  static constexpr int ODD = F == 9 ? 3 : (F == 25 ? 5 : F);
  static constexpr int NPOW = A / 3 + (A % 3 ? 1 : 0);
  static constexpr int NP = NODD + NPOW;
  __host__ __device__ static constexpr int radix(int i) {
    if (i < NODD) return ODD;
    const int k = i - NODD;  // k-th power-of-two pass
    return k < A / 3 ? 8 : (A % 3 == 2 ? 4 : 2);
  }
  __host__ __device__ static constexpr int ns(int i) { return i == 0 ? 1 : ns(i - 1) * radix(i - 1); }
};

template <class CP, int I, int IEND, bool INV, int N, int ROWS>
__device__ __forceinline__ void middle_passes(double2* s, const double2* __restrict__ twN) {
  if constexpr (I < IEND) {
    stockham_pass_x<CP::radix(I), INV, N, CP::ns(I), ROWS>(s, twN);
    middle_passes<CP, I + 1, IEND, INV, N, ROWS>(s, twN);
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft_any(double2* v) {
  if constexpr ((R & (R - 1)) == 0) dft_reg<R, INV>(v);
  else dft_odd<R, INV>(v);
}

template <int A, int F, bool INV>
__global__ void __launch_bounds__(FFT_T, 4)
fft_colx2_kernel(double2* __restrict__ buf, int64_t ustride, UnitTable ut, FftGeom g, int mask_input,
                 const double2* __restrict__ ftab, const double2* __restrict__ chirp) {
  extern __shared__ double2 s[];
  using CP = ColPasses<F, A>;
  constexpr int P1 = F << A;
  constexpr int P2 = 2048;
  constexpr int C = fft_col_ctas_cols(P1, 2048);
  constexpr int E = C * P1;
  constexpr int rstride = rstride_x(P1);
  static_assert(CP::NP >= 2, "hand-off variant needs distinct first and last passes");
  const int u = blockIdx.y;
  const int c0 = blockIdx.x * C;
  const int lat = ut.lat[u];
  const int64_t m = ut.m[lat];
  double2* ub = buf + (int64_t)u * ustride;
  const double2* twN = ftab + g.off_p1;

  {  // first pass (Ns = 1, no twiddles) from global memory
    constexpr int R0 = CP::radix(0);
    constexpr int per = P1 / R0;
    constexpr int NB = C * per;
    constexpr int BPT = (NB + FFT_T - 1) / FFT_T;
    double2 v[BPT][R0];
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      const int b = threadIdx.x + q * FFT_T;
      const int c = b % C, j = b / C;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        v[q][r] = make_double2(0.0, 0.0);
        if (NB % FFT_T == 0 || b < NB) {
          const int64_t n = (int64_t)(j + r * per) * P2 + c0 + c;
          if (INV || !mask_input || n < m) v[q][r] = ub[n];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      const int b = threadIdx.x + q * FFT_T;
      if (NB % FFT_T == 0 || b < NB) {
        const int c = b % C, j = b / C;
        dft_any<R0, INV>(v[q]);
#pragma unroll
        for (int r = 0; r < R0; ++r) s[c * rstride + Tile<2048>::pad(j * R0 + r)] = v[q][out_slot<R0>(r)];
      }
    }
    __syncthreads();
  }
  middle_passes<CP, 1, CP::NP - 1, INV, P1, C>(s, twN);
  {  // last pass (k = j) into registers, then twiddle / post-chirp and store
    constexpr int RL = CP::radix(CP::NP - 1);
    constexpr int NSL = CP::ns(CP::NP - 1);  // = P1 / RL
    constexpr int NB = C * NSL;
    constexpr int BPT = (NB + FFT_T - 1) / FFT_T;
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      const int b = threadIdx.x + q * FFT_T;
      if (NB % FFT_T == 0 || b < NB) {
        const int c = b % C, j = b / C;
        double2 v[RL];
#pragma unroll
        for (int r = 0; r < RL; ++r) v[r] = s[c * rstride + Tile<2048>::pad(j + r * NSL)];
        {  // w^{r j}, w = e^{-2 pi i / P1} (tstep = 1), as stockham_pass_x
          const double2 w1 = __ldg(&twN[j]);
          double2 w = w1;
#pragma unroll
          for (int r = 1; r < RL; ++r) {
            v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
            if (r + 1 < RL) w = cmul(w, w1);
          }
        }
        dft_any<RL, INV>(v);
        const int64_t n2 = c0 + c;
        if (!INV) {
          // output k1 = j + r NSL: e^{-2 pi i n2 k1 / P} by a recurrence over r
          double2 w = twP(g, ftab, n2 * (int64_t)j);
          const double2 step = twP(g, ftab, n2 * (int64_t)NSL);
#pragma unroll
          for (int r = 0; r < RL; ++r) {
            ub[(int64_t)(j + r * NSL) * P2 + n2] = cmul(v[out_slot<RL>(r)], w);
            if (r + 1 < RL) w = cmul(w, step);
          }
        } else {
          // post-chirp read from the lattice table, or (chirp == nullptr)
          // recomputed bit-identically: 16 B per output point less traffic
          const double2* ch = chirp ? chirp + ut.off[lat] : nullptr;
          const uint64_t inv2m = ~0ull / (2 * (uint64_t)m);
#pragma unroll
          for (int r = 0; r < RL; ++r) {
            const int64_t n = (int64_t)(j + r * NSL) * P2 + n2;
            if (n < m) ub[n] = cmul(v[out_slot<RL>(r)], ch ? __ldg(&ch[n]) : chirp_at(n, m, inv2m));
          }
        }
      }
    }
  }
}

static bool colx2_enabled() {
  static const bool v = [] {
    const char* e = getenv("SFFT_B200_FFT_COLX2");
    return !(e && strcmp(e, "0") == 0);
  }();
  return v;
}

template <int A, int F>
static int launch_colx_t(bool inv, const FftGeom& g, dim3 grid, cudaStream_t st, double2* buf, int64_t us,
                         const UnitTable& ut, int mask, const double2* ftab, const double2* chirp) {
  constexpr int P1 = F << A;
  const size_t sm = (size_t)fft_col_ctas_cols(P1, 2048) * rstride_x(P1) * sizeof(double2);
  if constexpr (ColPasses<F, A>::NP >= 2) {
    if (colx2_enabled()) {
      const void* fn2 = inv ? (const void*)fft_colx2_kernel<A, F, true> : (const void*)fft_colx2_kernel<A, F, false>;
      cudaError_t e2 = set_smem_once(fn2, sm);
      if (e2 != cudaSuccess) return (int)e2;
      if (inv) fft_colx2_kernel<A, F, true><<<grid, FFT_T, sm, st>>>(buf, us, ut, g, mask, ftab, chirp);
      else fft_colx2_kernel<A, F, false><<<grid, FFT_T, sm, st>>>(buf, us, ut, g, mask, ftab, chirp);
      SFFT_CHECK_LAUNCH();
      return 0;
    }
  }
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
    case 1:  // power-of-two columns of >= 16 (two or more passes) in 2048-element tiles
      if (g.a1 < 4) return -22;
      return dispatch_a<1, 4>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    case 3: return dispatch_a<3, 0>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    case 5: return dispatch_a<5, 0>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    case 7: return dispatch_a<7, 0>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    case 9: return dispatch_a<9, 0>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    case 25: return dispatch_a<25, 0>(g.a1, inv, g, grid, st, buf, ustride, ut, mask_input, ftab, chirp);
    default: return -22;
  }
}

}  // namespace sfft
