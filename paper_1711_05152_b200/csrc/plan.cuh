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

// Power-of-two FFT geometry: P = P1 * P2, P2 = 2^min(11, p) (tiles of 2048)
// for p <= 22, P2 = 4096 (tiles of 4096) for p = 23, 24.
struct FftGeom {
  int p, p1, p2, P1, P2, qlo, nlo;
  int te;  // shared-memory tile (elements): 2048 for p <= 22, 4096 above
  int64_t P;
  int64_t off_p1, off_p2, off_lo, off_hi, table_len;
};

__host__ __device__ inline FftGeom fft_geom(int p) {
  FftGeom g;
  g.p = p;
  g.te = p <= 22 ? 2048 : 4096;
  const int ptile = p <= 22 ? 11 : 12;
  g.p2 = p < ptile ? p : ptile;
  g.p1 = p - g.p2;
  g.P1 = 1 << g.p1;
  g.P2 = 1 << g.p2;
  g.P = (int64_t)1 << p;
  g.qlo = (p + 1) / 2;
  g.nlo = 1 << g.qlo;
  g.off_p1 = 0;
  g.off_p2 = g.P1;
  g.off_lo = g.P1 + g.P2;
  g.off_hi = g.off_lo + g.nlo;
  g.table_len = g.off_hi + ((int64_t)1 << (p - g.qlo));
  return g;
}

int launch_fft_tables(int p, double2* out, cudaStream_t st);
int launch_lattice_tables(const LatTable& lt, double2* tw, double2* chirp, cudaStream_t st);
int launch_bhat(const LatTable& lt, const double2* chirp, double2* bhat, int p,
                const double2* ftab, cudaStream_t st);
int launch_bluestein(double2* buf, const UnitTable& ut, int p, const double2* ftab,
                     const double2* bhat, const double2* chirp, cudaStream_t st);

}  // namespace sfft
