// Launch-parameter structs passed BY VALUE to the kernels (CUDA >= 12.1 allows
// 32 KB of kernel parameters), so lattice metadata never needs an H2D copy or
// a host synchronisation.
#pragma once
#include "common.cuh"

#define SFFT_UMAX 256        // (iteration, lattice) units per launch
#define SFFT_ZMAX 4096       // L * d generating-vector entries per launch

namespace sfft {

// Lattices of one MR1L step: sizes, reciprocals, table offsets, z vectors.
struct LatTable {
  int nlat;
  int d;                      // length of each z (the candidates' dimension t+1)
  int i32;                    // residues fit the int32 path (d * kmax * M < 2^31)
  int64_t m[SFFT_LMAX];
  double inv_m[SFFT_LMAX];
  int64_t off[SFFT_LMAX];     // offset of lattice l in the per-lattice tw/chirp tables
  uint32_t off32[SFFT_LMAX];  // int32 path: M_l * d * kmax (non-negative shift, multiple of M_l)
  uint32_t mu32[SFFT_LMAX];   // int32 path: floor((2^32 - 1) / M_l)
  int32_t z[SFFT_ZMAX];       // z[l * d + c], canonicalised into [0, M_l)
};

// residue of candidate k on lattice l of a LatTable (every exact mode)
#define SFFT_RES(DM, FAST, k, lt, l)                                                       \
  residue<DM, FAST>(k, (lt).d, (lt).z + (l) * (lt).d, (lt).m[l], (lt).inv_m[l], (lt).i32, \
                    (lt).off32[l], (lt).mu32[l])

// (iteration, lattice) work units of one step.
struct UnitTable {
  int nunits;
  int nlat;
  int lat[SFFT_UMAX];
  int it[SFFT_UMAX];
  int64_t m[SFFT_LMAX];
  int64_t off[SFFT_LMAX];
};

// row of the all-gathered per-unit buffer holding global unit u = it * L + l
struct RowMap {
  int row[SFFT_UMAX];
};

// Bluestein FFT geometry: P = P1 * P2.
//   P <= 2048          : one row (P1 = 1, P2 = P), power of two;
//   2^11 < P <= 2^22   : P2 = 2048 (tiles of 2048), P1 = f * 2^a <= 2048 with
//                        f in {1, 3, 5, 7, 9, 25} (mixed-radix column passes):
//                        P within 1.33x (mean 1.08x) of 2M - 1 instead of 2x;
//   P = 2^23, 2^24     : P2 = 4096 (tiles of 4096), P1 = 2^11, 2^12.
// Twiddles e^{-2 pi i m / P} come from a two-level table: m = hi * nlo + lo.
__host__ __device__ inline bool fft_odd_ok(int64_t f) {
  return f == 1 || f == 3 || f == 5 || f == 7 || f == 9 || f == 25;
}

struct FftGeom {
  int valid;
  int a1, f1;  // P1 = f1 * 2^a1
  int p2, P1, P2, qlo, nlo;
  int te;  // shared-memory tile (elements): 2048 for P <= 2^22, 4096 above
  int64_t P, nhi;
  int64_t off_p1, off_p2, off_lo, off_hi, table_len;
};

__host__ __device__ inline FftGeom fft_geom(int64_t P) {
  FftGeom g;
  g.valid = 0;
  g.a1 = g.f1 = g.p2 = g.P1 = g.P2 = g.qlo = g.nlo = g.te = 0;
  g.P = P;
  g.nhi = g.off_p1 = g.off_p2 = g.off_lo = g.off_hi = g.table_len = 0;
  if (P < 16 || P > ((int64_t)1 << 24)) return g;
  int64_t odd = P;
  int e = 0;
  while (!(odd & 1)) { odd >>= 1; ++e; }
  if (odd == 1) {
    g.te = e <= 22 ? 2048 : 4096;
    const int ptile = e <= 22 ? 11 : 12;
    g.p2 = e < ptile ? e : ptile;
    g.a1 = e - g.p2;
    g.f1 = 1;
  } else {
    if (e < 11 || !fft_odd_ok(odd) || (odd << (e - 11)) > 2048) return g;
    g.te = 2048;
    g.p2 = 11;
    g.a1 = e - 11;
    g.f1 = (int)odd;
  }
  g.P1 = g.f1 << g.a1;
  g.P2 = 1 << g.p2;
  int lg = 0;
  while (((int64_t)1 << lg) < P) ++lg;
  g.qlo = (lg + 1) / 2;
  g.nlo = 1 << g.qlo;
  g.nhi = (P + g.nlo - 1) >> g.qlo;
  g.off_p1 = 0;
  g.off_p2 = g.P1;
  g.off_lo = g.P1 + g.P2;
  g.off_hi = g.off_lo + g.nlo;
  g.table_len = g.off_hi + g.nhi;
  g.valid = 1;
  return g;
}

// Smallest supported P >= 2 m_max - 1 (>= 16); -1 above 2^24.  pow2_only:
// powers of two only (the previous geometry, for comparisons).
inline int64_t fft_choose_size(int64_t m_max, bool pow2_only) {
  const int64_t need = 2 * m_max - 1 > 16 ? 2 * m_max - 1 : 16;
  if (need > ((int64_t)1 << 24)) return -1;
  int64_t best = 16;
  while (best < need) best <<= 1;
  if (pow2_only || need <= 2048) return best;
  const int fs[5] = {3, 5, 7, 9, 25};
  for (int i = 0; i < 5; ++i)
    for (int64_t p1 = fs[i]; p1 <= 2048; p1 <<= 1)
      if (p1 * 2048 >= need) {
        if (p1 * 2048 < best) best = p1 * 2048;
        break;
      }
  return best;
}

// columns per CTA of a column pass of length P1 in a tile of TE elements
__host__ __device__ constexpr int fft_col_ctas_cols(int P1, int TE) {
  int c = 1;
  while (2 * c * P1 <= TE) c *= 2;
  return c;
}

int launch_fft_tables(const FftGeom& g, double2* out, cudaStream_t st);
int launch_lattice_tables(const LatTable& lt, double2* tw, double2* chirp, cudaStream_t st);
int launch_bhat(const LatTable& lt, const double2* chirp, double2* bhat, const FftGeom& g,
                const double2* ftab, cudaStream_t st);
int launch_bluestein(double2* buf, const UnitTable& ut, const FftGeom& g, const double2* ftab,
                     const double2* bhat, const double2* chirp, cudaStream_t st);
// mixed-radix column pass (f1 > 1, tiles of 2048), fft_mixed.cu
int launch_colx(bool inv, const FftGeom& g, dim3 grid, cudaStream_t st, double2* buf, int64_t ustride,
                const UnitTable& ut, int mask_input, const double2* ftab, const double2* chirp);

}  // namespace sfft
