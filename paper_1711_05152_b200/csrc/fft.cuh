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
#include "plan.cuh"

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

// Stockham twiddles of one radix-R butterfly: v[r] *= w^r (conjugate if INV),
// w = twN[k * tstep]; w^r for r < R from two table entries (w^1, w^4): few
// live registers
template <int R, bool INV>
__device__ __forceinline__ void twiddle_reg(double2* v, int k, int tstep, const double2* __restrict__ twN) {
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
    v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
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
      if (Ns > 1) twiddle_reg<R, INV>(v[q], k, tstep, twN);
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

// ---------------------------------------------------------------------------
// Mixed-radix building blocks (column passes of length P1 = f * 2^a, f odd in
// {3, 5, 7, 9, 25}): odd-radix DFTs in registers and a Stockham pass for any
// radix over a tile of E elements (E = rows * N <= 2048).

// cos / sin of 2 pi m / R for m <= (R - 1) / 2
template <int R>
__device__ __forceinline__ double cos2pi(int m) {
  if constexpr (R == 3) return -0.5;
  else if constexpr (R == 5) return m == 1 ? 0.30901699437494742410 : -0.80901699437494742410;
  else return m == 1 ? 0.62348980185873353053 : (m == 2 ? -0.22252093395631440429 : -0.90096886790241912624);
}
template <int R>
__device__ __forceinline__ double sin2pi(int m) {
  if constexpr (R == 3) return 0.86602540378443864676;
  else if constexpr (R == 5) return m == 1 ? 0.95105651629515357212 : 0.58778525229247312917;
  else return m == 1 ? 0.78183148246802980871 : (m == 2 ? 0.97492791218182360702 : 0.43388373911755812048);
}

// Odd-radix DFT in registers, natural order in and out:
// X_k = sum_j v_j e^{-+2 pi i j k / R} via the symmetric pairs a_j = v_j + v_{R-j},
// b_j = v_j - v_{R-j}:  X_k, X_{R-k} = v_0 + sum_j cos(2pi jk/R) a_j -+ i sum_j sin(2pi jk/R) b_j.
template <int R, bool INV>
__device__ __forceinline__ void dft_odd(double2* v) {
  constexpr int H = (R - 1) / 2;
  double2 a[H], b[H];
#pragma unroll
  for (int j = 0; j < H; ++j) {
    a[j] = cadd(v[j + 1], v[R - 1 - j]);
    b[j] = csub(v[j + 1], v[R - 1 - j]);
  }
  const double2 x0 = v[0];
  double2 sum = x0;
#pragma unroll
  for (int j = 0; j < H; ++j) sum = cadd(sum, a[j]);
  v[0] = sum;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double2 re = x0, im = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      int m = (j * k) % R;
      const double sg = m > H ? -1.0 : 1.0;  // sin(2 pi (R - m) / R) = -sin(2 pi m / R)
      if (m > H) m = R - m;
      const double c = cos2pi<R>(m), sn = sg * sin2pi<R>(m);
      re = make_double2(fma(c, a[j - 1].x, re.x), fma(c, a[j - 1].y, re.y));
      im = make_double2(fma(sn, b[j - 1].x, im.x), fma(sn, b[j - 1].y, im.y));
    }
    // forward: X_k = re - i im, X_{R-k} = re + i im; inverse: signs swapped
    const double2 mi = make_double2(im.y, -im.x);  // -i * im
    v[k] = INV ? csub(re, mi) : cadd(re, mi);
    v[R - k] = INV ? cadd(re, mi) : csub(re, mi);
  }
}

template <int R>
__device__ __forceinline__ constexpr int out_slot(int r) {
  return (R & (R - 1)) == 0 ? bitrev_small(r, Log2<R>::v) : r;
}

// Row stride of the mixed-radix column tiles: the padded length made odd, so
// the rows of consecutive columns start in different 16-byte bank groups (the
// column-fastest first-pass stores and last-pass loads of C = 8 columns were
// 2-way bank conflicts with the even stride of N = 200: 226)
__host__ __device__ constexpr int rstride_x(int n) { return Tile<2048>::rstride(n) | 1; }

// One Stockham pass of radix R (any R <= 8) over ROWS rows of length N in
// shared memory (E = ROWS * N elements); NS = product of the radices already
// applied.  All sizes are compile-time (divisions become multiplies); the
// twiddles w^{r k} (w = e^{-2 pi i / (NS R)}) are powers of one table entry.
template <int R, bool INV, int N, int NS, int ROWS>
__device__ __forceinline__ void stockham_pass_x(double2* s, const double2* __restrict__ twN) {
  constexpr int E = ROWS * N;
  constexpr int BPT = (E / R + FFT_T - 1) / FFT_T;
  constexpr int per_row = N / R;
  constexpr int nb = ROWS * per_row;
  constexpr int tstep = N / (NS * R);
  constexpr int rstride = rstride_x(N);
  double2 v[BPT][R];
  int obase[BPT];
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    const int b = threadIdx.x + q * FFT_T;
    obase[q] = -1;
    if (nb % FFT_T == 0 || b < nb) {
      const int row = b / per_row;
      const int j = b - row * per_row;
      const int k = j % NS;
      const int base = row * rstride;
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = s[base + Tile<2048>::pad(j + r * per_row)];
      if constexpr (NS > 1) {
        const double2 w1 = __ldg(&twN[k * tstep]);
        double2 w = w1;
#pragma unroll
        for (int r = 1; r < R; ++r) {
          v[q][r] = INV ? cmulc(v[q][r], w) : cmul(v[q][r], w);
          if (r + 1 < R) w = cmul(w, w1);
        }
      }
      if constexpr ((R & (R - 1)) == 0) dft_reg<R, INV>(v[q]);
      else dft_odd<R, INV>(v[q]);
      obase[q] = base + (j - k) * R + k;  // row offset + unpadded index
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
        s[row * rstride + Tile<2048>::pad(idx0 + r * NS)] = v[q][out_slot<R>(r)];
    }
  }
  __syncthreads();
}

// power-of-two passes (radix 8, then 4/2) after the odd ones
template <int REM, bool INV, int N, int NS, int ROWS>
__device__ __forceinline__ void pow2_passes_x(double2* s, const double2* __restrict__ twN) {
  if constexpr (REM > 0) {
    constexpr int RB = REM >= 3 ? 3 : REM;
    stockham_pass_x<(1 << RB), INV, N, NS, ROWS>(s, twN);
    pow2_passes_x<REM - RB, INV, N, NS * (1 << RB), ROWS>(s, twN);
  }
}

// FFT of ROWS rows of length N = F * 2^A (natural order in/out)
template <int F, int A, bool INV, int ROWS>
__device__ __forceinline__ void block_fft_x(double2* s, const double2* __restrict__ twN) {
  constexpr int N = F << A;
  if constexpr (F == 9) {
    stockham_pass_x<3, INV, N, 1, ROWS>(s, twN);
    stockham_pass_x<3, INV, N, 3, ROWS>(s, twN);
  } else if constexpr (F == 25) {
    stockham_pass_x<5, INV, N, 1, ROWS>(s, twN);
    stockham_pass_x<5, INV, N, 5, ROWS>(s, twN);
  } else if constexpr (F > 1) {
    stockham_pass_x<F, INV, N, 1, ROWS>(s, twN);
  }
  pow2_passes_x<A, INV, N, F, ROWS>(s, twN);
}

// e^{-2 pi i m / P} (0 <= m < P) from the two-level table
__device__ __forceinline__ double2 twP(const FftGeom& g, const double2* __restrict__ tab, int64_t m) {
  const double2 lo = __ldg(&tab[g.off_lo + (m & (g.nlo - 1))]);
  const double2 hi = __ldg(&tab[g.off_hi + (m >> g.qlo)]);
  return cmul(hi, lo);
}

}  // namespace sfft
