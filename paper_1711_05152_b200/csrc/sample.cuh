#pragma once
#include "plan.cuh"

namespace sfft {

// anchor tails of the iterations in one launch: a[it * tail + c]
// anchor tails of the rb <= 8 iterations of a chunk (tail = d - t1 <= 63):
// by value in the launch parameters, so sized to what the engine passes
#define SFFT_ANCHOR_MAX 512
struct AnchorTable {
  int rb;
  int tail;
  double a[SFFT_ANCHOR_MAX];
};

// GEMM-factored polynomial sampling plan of one step (see sample.cu)
struct PolyPlan {
  int nunits;
  int s;
  int kind;  // 0: classic 64x64 tiles (sample.cu), 1: warp-specialised 64x128 tiles (sample_ws.cu)
  int bl;    // low bits of the two-level twiddle tables
  int ks;    // term slices per tile (K split)
  int kper;  // terms per slice (multiple of 16)
  int unit_lat[SFFT_UMAX];
  int unit_it[SFFT_UMAX];
  int tile_start[SFFT_UMAX + 1];  // CTA prefix over units (tiles * ks)
  int J1[SFFT_LMAX];
  int nt1[SFFT_LMAX];
  uint64_t mu[SFFT_LMAX];         // Barrett constants floor((2^64-1) / M_l)
  // kind 2: B operand panels (16 terms x 128 columns, 32 KB in MMA fragment
  // order) precomputed once per (lattice, column tile, 16-term chunk) at the
  // start of the sampling scratch: block panel_off[l] + tj2 * nchunk_total +
  // h / 16.  Independent of the K split and of the early-exit L (a prefix of
  // the L_max panels is the L panels).  Partial sums follow at partial_base.
  int nt2[SFFT_LMAX];
  int panel_off[SFFT_LMAX];
  int nchunk_total;
  int npanels;
  long long partial_base;
  long long flag_base;  // kind 2 with a K split: per-CTA publish flags (SFFT_WS_MAX_FLAGS u32)
};

#define SFFT_WS_MAX_FLAGS 1024

// B-spline test function: groups of (order, component slots)
struct BsplineSpec {
  int d;
  int ngroups;
  int order[8];
  int start[9];
  int comps[SFFT_DMAX];
  double scale[8];  // C_m * m
  // piecewise-polynomial form of the cardinal B-spline of order m on [0, m]:
  // piece iv (u in [iv, iv + 1)) is sum_k pc[bs_poff(m) + iv * m + k] t^k,
  // t = u - iv (filled by the host from the Cox-de Boor recursion)
  double pc[140];
};

__host__ __device__ constexpr int bs_poff(int m) { return (m - 1) * m * (2 * m - 1) / 6; }

int launch_poly_prepare(const int32_t* hf, const double2* coef, int s, int d, const LatTable& lt,
                        const PolyPlan& pp, const AnchorTable& at, double2* cprime, int32_t* rres,
                        int32_t* rj, cudaStream_t st);
int launch_sample_poly(const PolyPlan& pp, const LatTable& lt, const UnitTable& ut,
                       const double2* cprime, const int32_t* rres, const int32_t* rj,
                       const double2* tw, const double2* chirp, double2* buf, int64_t ustride,
                       bool apply_chirp, double2* scratch, int64_t pstride, int num_sms,
                       cudaStream_t st, bool panels_ready = false);
size_t sample_poly_smem(int bl, int64_t mmax);
size_t sample_poly_ws_smem(int bl, int64_t mmax);
int launch_bpanels(const PolyPlan& pp, const LatTable& lt, const int32_t* rj, const double2* tw, double* panels,
                   cudaStream_t st);
int launch_sample_poly_ws(const PolyPlan& pp, const LatTable& lt, const double2* cprime,
                          const int32_t* rres, const int32_t* rj, const double2* tw,
                          const double2* chirp, double2* buf, int64_t ustride, bool apply_chirp,
                          double2* part, int64_t pstride, double* panels, bool panels_ready,
                          unsigned* flags, bool* reduced, cudaStream_t st);
int launch_sample_bspline(const UnitTable& ut, const LatTable& lt, const BsplineSpec& bs,
                          const AnchorTable& at, const double2* chirp, double2* buf,
                          int64_t ustride, bool fast, bool apply_chirp, int num_sms,
                          cudaStream_t st);
int launch_finish_samples(const UnitTable& ut, const double2* chirp, double2* buf, int64_t ustride,
                          const double2* noise, int64_t nstride, const double* sigma, int num_sms,
                          cudaStream_t st);
int launch_finish_devnoise(const UnitTable& ut, const double2* chirp, double2* buf, int64_t ustride,
                           const double* norm2, double rel, double sigma, uint64_t seed,
                           uint64_t call_base, bool apply_chirp, int num_sms, cudaStream_t st);
int launch_unit_norm2(const UnitTable& ut, const double2* buf, int64_t ustride, double* out,
                      int num_sms, cudaStream_t st);
int launch_lattice_nodes(const LatTable& lt, int l, int d, const AnchorTable& at, int it,
                         double* pts, bool fast, cudaStream_t st);

// cardinal B-spline of order m (degree m-1) on knots 0..m, Cox-de Boor.
// Compile-time order: the triangle is fully unrolled in registers (a runtime
// order puts N[] in local memory and divides at every level); same
// arithmetic, same rounding as the runtime form.
template <int MO>
__device__ __forceinline__ double cardinal_bspline_t(double u) {
  if (!(u >= 0.0 && u <= (double)MO)) return 0.0;
  double N[MO + 1];
  int iv = (int)floor(u);
  if (iv >= MO) iv = MO - 1;
#pragma unroll
  for (int j = 0; j <= MO; ++j) N[j] = (j == iv) ? 1.0 : 0.0;
#pragma unroll
  for (int k = 2; k <= MO; ++k) {
    const double inv = 1.0 / (double)(k - 1);
#pragma unroll
    for (int j = 0; j <= MO - k; ++j) N[j] = ((u - j) * N[j] + ((double)(j + k) - u) * N[j + 1]) * inv;
  }
  return N[0];
}

__device__ __forceinline__ double cardinal_bspline(int m, double u) {
  switch (m) {
    case 1: return cardinal_bspline_t<1>(u);
    case 2: return cardinal_bspline_t<2>(u);
    case 3: return cardinal_bspline_t<3>(u);
    case 4: return cardinal_bspline_t<4>(u);
    case 5: return cardinal_bspline_t<5>(u);
    case 6: return cardinal_bspline_t<6>(u);
    default: return cardinal_bspline_t<7>(u);
  }
}


}  // namespace sfft
