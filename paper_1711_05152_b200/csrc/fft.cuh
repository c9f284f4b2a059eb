// In-shared-memory Stockham FFT building blocks shared by the Bluestein
// passes (fft.cu) and the line-detection kernel.
//
// A CTA of FFT_T = 256 threads owns a tile of TE complex128 elements,
// organised as `rows` independent transforms of length N = TE / rows.  Two
// tile shapes (template parameter TE):
//   TE = 2048: 8 values per thread, radix-8 passes, <= 64 registers, four
//              CTAs (32 warps) per SM — the default (P = 2^p, p <= 22);
//   TE = 4096: 16 values per thread, radix-16 passes, two CTAs per SM, for
//              the largest transforms (p = 23, 24).
// The passes are latency bound (shared-memory round trips, barriers): more
// resident CTAs overlap one CTA's DRAM phases with another's FFT passes.
#pragma once
#include "common.cuh"

namespace sfft {

constexpr int FFT_T = 256;

template <int TE>
struct Tile {
  static constexpr int E = TE;
  static constexpr int V = TE / FFT_T;           // values per thread and pass
  static constexpr int LV = V == 16 ? 4 : 3;     // log2 of the largest radix
  static constexpr int PADS = V == 16 ? 4 : 3;   // one padding slot per 2^PADS
  // padded shared-memory index of element i inside a row: the radix-V scatter
  // of the first pass (lane stride V) becomes bank-conflict free
  __device__ static __forceinline__ int pad(int i) { return i + (i >> PADS); }
  __host__ __device__ static constexpr int rstride(int n) { return n + (n >> PADS) + 1; }
};

// constant twiddles of the 16th roots of unity: e^{-2 pi i m / 16}, m < 8
__device__ __forceinline__ double2 tw16(int m, bool inv) {
  const double c1 = 0.92387953251128673848, s1 = 0.38268343236508977173;
  const double h = 0.70710678118654752440;
  double cr, ci;
  switch (m) {
    case 0: cr = 1.0; ci = 0.0; break;
    case 1: cr = c1; ci = -s1; break;
    case 2: cr = h; ci = -h; break;
    case 3: cr = s1; ci = -c1; break;
    case 4: cr = 0.0; ci = -1.0; break;
    case 5: cr = -s1; ci = -c1; break;
    case 6: cr = -h; ci = -h; break;
    default: cr = -c1; ci = -s1; break;
  }
  return make_double2(cr, inv ? -ci : ci);
}

template <bool INV>
__device__ __forceinline__ double2 twmul_const(double2 x, int m) {
  if (m == 0) return x;
  if (m == 4) return INV ? make_double2(-x.y, x.x) : make_double2(x.y, -x.x);
  return cmul(x, tw16(m, INV));
}

__host__ __device__ constexpr int bitrev_small(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}

template <int R>
struct Log2 { static constexpr int v = (R <= 1) ? 0 : 1 + Log2<R / 2>::v; };
template <>
struct Log2<1> { static constexpr int v = 0; };

// Radix-R DFT in registers (decimation in frequency): natural order in,
// X[k] left in v[bitrev(k)] (callers index the outputs through bitrev_small,
// a compile-time permutation, so no register shuffle is needed).
template <int R, bool INV>
__device__ __forceinline__ void dft_reg(double2* v) {
#pragma unroll
  for (int span = R / 2; span >= 1; span >>= 1) {
#pragma unroll
    for (int b = 0; b < R; b += 2 * span) {
#pragma unroll
      for (int q = 0; q < span; ++q) {
        double2 a = v[b + q], c = v[b + q + span];
        v[b + q] = cadd(a, c);
        v[b + q + span] = twmul_const<INV>(csub(a, c), q * (16 / (2 * span)));
      }
    }
  }
}

// One Stockham radix-R pass over `rows` rows of length N (all in smem).
// twN[m] = e^{-2 pi i m / N}, m < N (global, read-only).
template <int R, bool INV, int TE>
__device__ __forceinline__ void stockham_pass(double2* s, int rows, int rstride, int N, int Ns,
                                              const double2* __restrict__ twN) {
  constexpr int BPT = Tile<TE>::V / R;
  const int per_row = N / R;
  const int nb = rows * per_row;
  const int tstep = N / (Ns * R);
  double2 v[BPT][R];
  int obase[BPT];
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    const int b = threadIdx.x + q * FFT_T;
    obase[q] = -1;
    if (b < nb) {
      const int row = b / per_row;
      const int j = b - row * per_row;
      const int k = j & (Ns - 1);
      const int base = row * rstride;
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = s[base + Tile<TE>::pad(j + r * per_row)];
      if (Ns > 1) {
        // w^r for r < R from two table entries (w^1, w^4): few live registers
        const double2 w1 = __ldg(&twN[k * tstep]);
        double2 wl[4];
        wl[0] = make_double2(1.0, 0.0);
        wl[1] = w1;
        if (R > 2) { wl[2] = cmul(w1, w1); wl[3] = cmul(wl[2], w1); }
        double2 w4 = make_double2(1.0, 0.0);
        if (R > 4) w4 = __ldg(&twN[4 * k * tstep]);
        double2 wh = make_double2(1.0, 0.0);
#pragma unroll
        for (int r = 1; r < R; ++r) {
          if ((r & 3) == 0) wh = (r == 4) ? w4 : cmul(wh, w4);
          const double2 w = (r & 3) == 0 ? wh : ((r < 4) ? wl[r & 3] : cmul(wh, wl[r & 3]));
          v[q][r] = INV ? cmulc(v[q][r], w) : cmul(v[q][r], w);
        }
      }
      dft_reg<R, INV>(v[q]);
      obase[q] = row * rstride + ((j - k) * R + k);  // row offset + unpadded index
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    if (obase[q] >= 0) {
      const int b = threadIdx.x + q * FFT_T;
      const int row = b / per_row;
      const int idx0 = obase[q] - row * rstride;
#pragma unroll
      for (int r = 0; r < R; ++r)
        s[row * rstride + Tile<TE>::pad(idx0 + r * Ns)] = v[q][bitrev_small(r, Log2<R>::v)];
    }
  }
  __syncthreads();
}

// Full Stockham FFT of TE >> LOGN rows of length 2^LOGN (natural order
// in/out), fully unrolled at compile time: largest-radix passes first, one
// smaller pass last.
template <int LOGN, int DONE, bool INV, int TE>
__device__ __forceinline__ void fft_passes(double2* s, const double2* __restrict__ twN) {
  if constexpr (DONE < LOGN) {
    constexpr int REM = LOGN - DONE;
    constexpr int RB = REM >= Tile<TE>::LV ? Tile<TE>::LV : REM;
    stockham_pass<(1 << RB), INV, TE>(s, TE >> LOGN, Tile<TE>::rstride(1 << LOGN), 1 << LOGN, 1 << DONE, twN);
    fft_passes<LOGN, DONE + RB, INV, TE>(s, twN);
  }
}

template <int LOGN, bool INV, int TE>
__device__ __forceinline__ void block_fft(double2* s, const double2* __restrict__ twN) {
  fft_passes<LOGN, 0, INV, TE>(s, twN);
}

}  // namespace sfft
