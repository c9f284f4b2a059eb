// One-dimensional line detection of component t (reference detect.py:175-240:
// projected_line_coefficients + _select + union inside detect_component).
//
// Each of the r lines samples K_t points x = anchor with x_t = l / K_t.  For a
// sparse polynomial the sample is evaluated with an exact integer phase
//     p(x_l) = sum_h c''_h w_K^{(h_t l) mod K},  c''_h = c_h e^{2 pi i sum_{u != t} h_u a_u},
// then bins = DFT_K(samples) * (1/K), bin l <-> the k in [lo, hi] with
// k = l (mod K), and the line keeps the up-to-cap largest |coefficients| >=
// delta (ties: |c| desc, k asc).  Lines up to K = 1024 take one CTA each for
// sampling and for DFT + selection.  Longer lines (any K, SURVEY §8a-2 puts
// no limit on the box) are sampled by a tiled kernel with exact per-point
// phases; their DFT is the batched Bluestein path (transform.py:50-64) and
// line_bins_kernel maps the spectra to thresholded coefficients, the cap
// then being the exact row selection of the MR1L step (sfft_select_cap_rows).
#include "common.cuh"
#include "plan.cuh"
#include "lines.cuh"

namespace sfft {

constexpr int LT = 256;
constexpr int LCH = 512;  // terms per shared-memory chunk

// Grid (line, block of 32 points): each CTA evaluates 32 consecutive points
// of one line (8 warps split the terms, lane = point), so all lines and
// point blocks of a launch run side by side.  ``t`` >= 0: every line is of
// component t; t < 0: line g is of component g / rpc (all components'
// lines in one launch, anchors la.a + g * d).  Each point's sum runs in the
// same order whatever the grid: terms in chunks of LCH, warp w taking terms
// w, w + 8, ..., the 8 warp sums added in warp order.
__global__ void __launch_bounds__(LT)
line_sample_poly_kernel(const int32_t* __restrict__ hf, const double2* __restrict__ coef, int s,
                        int d, int t, int rpc, int K, LineAnchors la, double2* __restrict__ values) {
  __shared__ double2 cs[LCH];
  __shared__ int es[LCH];
  __shared__ double2 wk[1024];
  __shared__ double2 part[8][32];
  const int line = blockIdx.x;
  const int tc = t >= 0 ? t : line / rpc;
  const double* a = la.a + line * d;
  for (int q = threadIdx.x; q < K; q += LT) {
    double sn, c;
    sincospi(2.0 * (double)q / (double)K, &sn, &c);
    wk[q] = make_double2(c, sn);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int l0 = blockIdx.y * 32;
  const int l = l0 + lane;
  double2 acc = make_double2(0.0, 0.0);
  for (int h0 = 0; h0 < s; h0 += LCH) {
    __syncthreads();
    for (int q = threadIdx.x; q < LCH; q += LT) {
      const int h = h0 + q;
      double2 cc = make_double2(0.0, 0.0);
      int e = 0;
      if (h < s) {
        double ph = 0.0;
        for (int u = 0; u < d; ++u)
          if (u != tc) ph += (double)hf[(int64_t)u * s + h] * a[u];
        double sn, c;
        sincospi(2.0 * ph, &sn, &c);
        cc = cmul(coef[h], make_double2(c, sn));
        e = (int)mod_slow((int64_t)hf[(int64_t)tc * s + h], K);
      }
      cs[q] = cc;
      es[q] = e;
    }
    __syncthreads();
    if (l < K) {
      for (int q = w; q < LCH && h0 + q < s; q += 8) {
        const int idx = (int)(((int64_t)es[q] * l) % K);
        const double2 tw = wk[idx];
        const double2 cc = cs[q];
        acc.x = fma(cc.x, tw.x, acc.x);
        acc.x = fma(-cc.y, tw.y, acc.x);
        acc.y = fma(cc.x, tw.y, acc.y);
        acc.y = fma(cc.y, tw.x, acc.y);
      }
    }
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && l < K) {
    double2 t2 = part[0][lane];
    for (int q = 1; q < 8; ++q) t2 = cadd(t2, part[q][lane]);
    values[(int64_t)line * K + l] = t2;
  }
}

// K > 1024: grid (line, block of LT points); twiddles e^{2 pi i idx / K} with
// the exact integer phase idx = (e l) mod K evaluated directly
__global__ void __launch_bounds__(LT)
line_sample_poly_big_kernel(const int32_t* __restrict__ hf, const double2* __restrict__ coef, int s,
                            int d, int t, int K, LineAnchors la, double2* __restrict__ values) {
  __shared__ double2 cs[LCH];
  __shared__ int es[LCH];
  const int line = blockIdx.y;
  const double* a = la.a + line * d;
  const int l = blockIdx.x * LT + threadIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  for (int h0 = 0; h0 < s; h0 += LCH) {
    __syncthreads();
    for (int q = threadIdx.x; q < LCH; q += LT) {
      const int h = h0 + q;
      double2 cc = make_double2(0.0, 0.0);
      int e = 0;
      if (h < s) {
        double ph = 0.0;
        for (int u = 0; u < d; ++u)
          if (u != t) ph += (double)hf[(int64_t)u * s + h] * a[u];
        double sn, c;
        sincospi(2.0 * ph, &sn, &c);
        cc = cmul(coef[h], make_double2(c, sn));
        e = (int)mod_slow((int64_t)hf[(int64_t)t * s + h], K);
      }
      cs[q] = cc;
      es[q] = e;
    }
    __syncthreads();
    if (l < K) {
      for (int q = 0; q < LCH && h0 + q < s; ++q) {
        const int64_t idx = ((int64_t)es[q] * l) % K;
        double sn, c;
        sincospi(2.0 * (double)idx / (double)K, &sn, &c);
        const double2 cc = cs[q];
        acc.x = fma(cc.x, c, acc.x);
        acc.x = fma(-cc.y, sn, acc.x);
        acc.y = fma(cc.x, sn, acc.y);
        acc.y = fma(cc.y, c, acc.y);
      }
    }
  }
  if (l < K) values[(int64_t)line * K + l] = acc;
}

// K > 1024: spectra (row i at spec + i * P, the unnormalised forward DFT of
// line i) -> coefficient of k = lo + q is bin (k mod K) * (1/K), threshold
// flag and per-line survivor count (integer atomics: order-free, exact)
__global__ void line_bins_kernel(const double2* __restrict__ spec, int64_t P, int K, int64_t lo, double delta,
                                 double2* __restrict__ coefs, uint8_t* __restrict__ keep,
                                 int32_t* __restrict__ counts) {
  const int line = blockIdx.y;
  const double invk = 1.0 / (double)K;
  int cnt = 0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < K; q += gridDim.x * blockDim.x) {
    const int bin = (int)mod_slow(lo + q, K);
    const double2 x = spec[(int64_t)line * P + bin];
    const double2 c = make_double2(x.x * invk, x.y * invk);
    coefs[(int64_t)line * K + q] = c;
    const uint8_t kf = hypot(c.x, c.y) >= delta ? 1 : 0;
    keep[(int64_t)line * K + q] = kf;
    cnt += kf;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&counts[line], cnt);
}

// DFT of each line, bin mapping, threshold and cap ranking
__global__ void __launch_bounds__(LT)
line_select_kernel(const double2* __restrict__ values, int K, int64_t lo, int cap, double delta,
                   double2* __restrict__ coefs, uint8_t* __restrict__ keep) {
  __shared__ double2 v[1024];
  __shared__ double2 wk[1024];
  __shared__ double mg[1024];
  __shared__ uint8_t pre[1024];
  __shared__ int red[32];
  const int line = blockIdx.x;
  for (int q = threadIdx.x; q < K; q += LT) {
    double sn, c;
    sincospi(2.0 * (double)q / (double)K, &sn, &c);
    wk[q] = make_double2(c, -sn);  // forward: e^{-2 pi i q / K}
    v[q] = values[(int64_t)line * K + q];
  }
  __syncthreads();
  const double invk = 1.0 / (double)K;
  // coefficient of k = lo + q is bin (k mod K)
  int cnt = 0;
  for (int q = threadIdx.x; q < K; q += LT) {
    const int64_t k = lo + q;
    const int bin = (int)mod_slow(k, K);
    double2 acc = make_double2(0.0, 0.0);
    for (int l = 0; l < K; ++l) {
      const int idx = (int)(((int64_t)bin * l) % K);
      acc = cadd(acc, cmul(v[l], wk[idx]));
    }
    const double2 c = make_double2(acc.x * invk, acc.y * invk);
    coefs[(int64_t)line * K + q] = c;
    const double m = hypot(c.x, c.y);
    mg[q] = m;
    pre[q] = (m >= delta) ? 1 : 0;
    cnt += pre[q];
  }
  __syncthreads();
  const int total = block_sum(cnt, red);
  __shared__ int tot_s;
  if (threadIdx.x == 0) tot_s = total;
  __syncthreads();
  const int tot = tot_s;
  for (int q = threadIdx.x; q < K; q += LT) {
    uint8_t kf = pre[q];
    if (kf && tot > cap) {
      int rank = 0;
      const double m = mg[q];
      for (int q2 = 0; q2 < K; ++q2)
        if (pre[q2] && (mg[q2] > m || (mg[q2] == m && q2 < q))) ++rank;
      kf = rank < cap ? 1 : 0;
    }
    keep[(int64_t)line * K + q] = kf;
  }
}

int launch_line_sample_poly(const int32_t* hf, const double2* coef, int s, int d, int t, int K,
                            const LineAnchors& la, int r, double2* values, cudaStream_t st) {
  if (K < 1 || r <= 0 || r > 65535) return -22;
  if (K > 1024) {
    if (t < 0) return -22;
    line_sample_poly_big_kernel<<<dim3((K + LT - 1) / LT, r), LT, 0, st>>>(hf, coef, s, d, t, K, la, values);
  } else {
    line_sample_poly_kernel<<<dim3(r, (K + 31) / 32), LT, 0, st>>>(hf, coef, s, d, t, r, K, la, values);
  }
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_line_sample_poly_all(const int32_t* hf, const double2* coef, int s, int d, int K,
                                const LineAnchors& la, int r, double2* values, cudaStream_t st) {
  if (K < 1 || K > 1024 || r <= 0 || (int64_t)r * d > 65535) return -22;
  line_sample_poly_kernel<<<dim3(r * d, (K + 31) / 32), LT, 0, st>>>(hf, coef, s, d, -1, r, K, la, values);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_line_select(const double2* values, int r, int K, int64_t lo, int cap, double delta,
                       double2* coefs, uint8_t* keep, cudaStream_t st) {
  if (K > 1024 || r <= 0) return -22;
  line_select_kernel<<<r, LT, 0, st>>>(values, K, lo, cap, delta, coefs, keep);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_line_bins(const double2* spec, int64_t P, int r, int K, int64_t lo, double delta, double2* coefs,
                     uint8_t* keep, int32_t* counts, int num_sms, cudaStream_t st) {
  if (K < 1 || r <= 0 || r > 65535 || P < K) return -22;
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)r, st);
  if (e != cudaSuccess) return (int)e;
  int bx = (K + 255) / 256;
  const int cap = (num_sms * 8 + r - 1) / r;
  if (bx > cap) bx = cap > 0 ? cap : 1;
  line_bins_kernel<<<dim3(bx, r), 256, 0, st>>>(spec, P, K, lo, delta, coefs, keep, counts);
  SFFT_CHECK_LAUNCH();
  return 0;
}

}  // namespace sfft
