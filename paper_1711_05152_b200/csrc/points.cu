// Oracle evaluation at arbitrary points (the device-oracle descriptors'
// __call__, reference testbed.py:60-73 / 116-127 / 232-244).  Used for line
// samples of non-polynomial oracles and by users calling an oracle directly;
// lattice nodes use the fused kernels in sample.cu.
#include "common.cuh"
#include "plan.cuh"
#include "sample.cuh"

namespace sfft {

constexpr int PCH = 256;

// p(x) = sum_h c_h e^{2 pi i h.x}; phase accumulated in float64 per point
__global__ void __launch_bounds__(256)
eval_poly_points_kernel(const double* __restrict__ pts, int64_t n, int d,
                        const int32_t* __restrict__ hf, const double2* __restrict__ coef, int s,
                        double2* __restrict__ out) {
  __shared__ double2 cs[PCH];
  __shared__ int32_t fs[PCH * 8];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  const int dc = d < 8 ? d : 8;  // components staged in shared memory
  for (int h0 = 0; h0 < s; h0 += PCH) {
    __syncthreads();
    for (int q = threadIdx.x; q < PCH; q += blockDim.x) {
      const int h = h0 + q;
      cs[q] = h < s ? coef[h] : make_double2(0.0, 0.0);
      for (int c = 0; c < dc; ++c) fs[c * PCH + q] = h < s ? hf[(int64_t)c * s + h] : 0;
    }
    __syncthreads();
    if (i < n) {
      const int hn = (s - h0) < PCH ? (s - h0) : PCH;
      for (int q = 0; q < hn; ++q) {
        double ph = 0.0;
        for (int c = 0; c < d; ++c) {
          const int32_t k = c < 8 ? fs[c * PCH + q] : hf[(int64_t)c * s + h0 + q];
          ph = fma(pts[i * d + c], (double)k, ph);
        }
        double sn, cn;
        sincospi(2.0 * ph, &sn, &cn);
        const double2 cc = cs[q];
        acc.x = fma(cc.x, cn, acc.x);
        acc.x = fma(-cc.y, sn, acc.x);
        acc.y = fma(cc.x, sn, acc.y);
        acc.y = fma(cc.y, cn, acc.y);
      }
    }
  }
  if (i < n) out[i] = acc;
}

__global__ void eval_bspline_points_kernel(const double* __restrict__ pts, int64_t n, BsplineSpec bs,
                                           double2* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double total = 0.0;
    for (int g = 0; g < bs.ngroups; ++g) {
      const int m = bs.order[g];
      double term = 1.0;
      for (int q = bs.start[g]; q < bs.start[g + 1]; ++q) {
        double x = pts[i * bs.d + bs.comps[q]];
        x = x - floor(x);  // np.mod(x, 1.0) for finite x
        if (x >= 1.0) x = 0.0;
        term = term * (bs.scale[g] * cardinal_bspline(m, (double)m * x));
      }
      total += term;
    }
    out[i] = make_double2(total, 0.0);
  }
}

// x += scale * e (complex), the NoisyOracle update of testbed.py:104-106
__global__ void add_noise_kernel(double2* __restrict__ x, const double2* __restrict__ e, int64_t n,
                                 double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = x[i], w = e[i];
    x[i] = make_double2(v.x + scale * w.x, v.y + scale * w.y);
  }
}

int launch_eval_poly_points(const double* pts, int64_t n, int d, const int32_t* hf,
                            const double2* coef, int s, double2* out, cudaStream_t st) {
  if (n == 0) return 0;
  eval_poly_points_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pts, n, d, hf, coef, s, out);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// The points of r anchored axis lines of every component t < d (K points
// each, x_t = l / K): row (g K + l), g = t r + i, is anchors[g] with
// component t = g / r replaced by l / K (the host's np.arange(K) / K).
__global__ void line_points_kernel(const double* __restrict__ anchors, int d, int r, int K,
                                   double* __restrict__ pts) {
  const int64_t total = (int64_t)d * r * K * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / d;
    const int c = (int)(e - row * d);
    const int64_t g = row / K;
    const int l = (int)(row - g * K);
    pts[e] = c == (int)(g / r) ? (double)l / (double)K : anchors[g * d + c];
  }
}

int launch_line_points(const double* anchors, int d, int r, int K, double* pts, int num_sms, cudaStream_t st) {
  const int64_t total = (int64_t)d * r * K * d;
  if (total <= 0) return 0;
  int64_t want = (total + 255) / 256, cap = (int64_t)num_sms * 8;
  line_points_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(anchors, d, r, K, pts);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_eval_bspline_points(const double* pts, int64_t n, const BsplineSpec& bs, double2* out,
                               int num_sms, cudaStream_t st) {
  if (n == 0) return 0;
  int64_t want = (n + 255) / 256, cap = (int64_t)num_sms * 8;
  eval_bspline_points_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(pts, n, bs, out);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_add_noise(double2* x, const double2* e, int64_t n, double scale, int num_sms,
                     cudaStream_t st) {
  if (n == 0) return 0;
  int64_t want = (n + 255) / 256, cap = (int64_t)num_sms * 8;
  add_noise_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(x, e, n, scale);
  SFFT_CHECK_LAUNCH();
  return 0;
}

}  // namespace sfft
