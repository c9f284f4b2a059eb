#pragma once
#include "plan.cuh"

namespace sfft {

// full anchors of the lines in one launch: a[line * d + u]
struct LineAnchors {
  double a[2048];
};

int launch_line_sample_poly(const int32_t* hf, const double2* coef, int s, int d, int t, int K,
                            const LineAnchors& la, int r, double2* values, cudaStream_t st);
// the r lines of every component t < d in one launch (K <= 1024): line
// g = t * r + i, anchors la.a[g * d ...], values row g
int launch_line_sample_poly_all(const int32_t* hf, const double2* coef, int s, int d, int K,
                                const LineAnchors& la, int r, double2* values, cudaStream_t st);
int launch_line_select(const double2* values, int r, int K, int64_t lo, int cap, double delta,
                       double2* coefs, uint8_t* keep, cudaStream_t st);
int launch_line_bins(const double2* spec, int64_t P, int r, int K, int64_t lo, double delta, double2* coefs,
                     uint8_t* keep, int32_t* counts, int num_sms, cudaStream_t st);

}  // namespace sfft
