// K1: sampling the signal at the nodes of the step's rank-1 lattices.
//
// Reference: detect.py:280-302 (_invert_candidates: nodes = lattice_nodes +
// anchor tail, one oracle call per lattice), lattice.py:505-508 (nodes
// x_j = (j z mod M) / M), testbed.py:116-127 (sparse polynomial oracle,
// p(x) = sum_h c_h e^{2 pi i h.x}), testbed.py:219-244 (B-spline oracle).
//
// Sparse polynomial at lattice nodes with exact integer phases:
//   p(x_j) = sum_h c'_h w^{(r_h j) mod M},   w = e^{2 pi i / M},
//   r_h = h_head . z mod M,  c'_h = c_h e^{2 pi i h_tail . anchor}.
// With j = j1 + J1 j2 the sum factors into a complex GEMM
//   v[j1 + J1 j2] = sum_h A[j1, h] B[h, j2],
//   A[j1, h] = c'_h w^{(r_h j1) mod M},  B[h, j2] = w^{((r_h J1 mod M) j2) mod M},
// whose operand tiles are generated on the fly from one twiddle table per
// lattice (L2-resident) and contracted with register-tiled DFMA (no tensor
// cores: FP64 tensor throughput equals DFMA throughput on B200).  The
// epilogue writes the Bluestein pre-chirped input x_j c_j directly (K1 -> K2
// fusion), so the length-M sample vector is never stored unchirped.
#include "common.cuh"
#include "plan.cuh"
#include "sample.cuh"

#include <cstdlib>
#include <cstring>

namespace sfft {

// c'[it, h] = c_h * e^{2 pi i sum_{c >= t1} h_c a[it, c - t1]}
__global__ void poly_rotate_kernel(const int32_t* __restrict__ hf, const double2* __restrict__ coef,
                                   int s, int d, int t1, AnchorTable at, double2* __restrict__ cprime) {
  const int it = blockIdx.y;
  const int tail = d - t1;
  for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < s; h += gridDim.x * blockDim.x) {
    double ph = 0.0;
    for (int c = 0; c < tail; ++c) ph += (double)hf[(int64_t)(t1 + c) * s + h] * at.a[it * tail + c];
    double2 cf = coef[h];
    if (tail > 0) {
      double sn, cs;
      sincospi(2.0 * ph, &sn, &cs);
      cf = cmul(cf, make_double2(cs, sn));
    }
    cprime[(int64_t)it * s + h] = cf;
  }
}

// (x mod m) for any x < 2^64 by Barrett reduction with mu = floor((2^64-1)/m):
// the quotient estimate is low by at most one, so one correction is exact.
// Integer pipe only (keeps the FP64 pipe for the contraction).
__device__ __forceinline__ uint32_t mod_barrett(uint64_t x, uint32_t m, uint64_t mu) {
  const uint64_t q = __umul64hi(x, mu);
  uint64_t r = x - q * (uint64_t)m;
  if (r >= m) r -= m;
  return (uint32_t)r;
}

// r_h = h_head . z_l mod M_l and r_h * J1_l mod M_l: exact for every M < 2^31
// (componentwise-reduced inner product as lattice.py:511-517; 32-bit
// remainder of the int32 component, Barrett reduction of each product)
__global__ void poly_residue_kernel(const int32_t* __restrict__ hf, int s, LatTable lt,
                                    PolyPlan pp, int32_t* __restrict__ rres, int32_t* __restrict__ rj) {
  const int l = blockIdx.y;
  const uint32_t m = (uint32_t)lt.m[l];
  const uint64_t mu = pp.mu[l];
  const int t1 = lt.d;
  for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < s; h += gridDim.x * blockDim.x) {
    uint32_t acc = 0;
    for (int c = 0; c < t1; ++c) {
      int32_t k = hf[(int64_t)c * s + h] % (int32_t)m;  // m <= 2^31 - 1 fits int32
      const uint32_t km = (uint32_t)(k < 0 ? k + (int32_t)m : k);
      acc += mod_barrett((uint64_t)km * (uint64_t)lt.z[l * t1 + c], m, mu);
      if (acc >= m) acc -= m;  // acc + x < 2m < 2^32
    }
    rres[(int64_t)l * s + h] = (int32_t)acc;
    rj[(int64_t)l * s + h] = (int32_t)mod_barrett((uint64_t)acc * (uint64_t)pp.J1[l], m, mu);
  }
}

constexpr int PT = 64;  // output tile edge (j1 and j2)
constexpr int KC = 16;  // terms per shared-memory stage
constexpr int SP_T = 256;  // threads per sampling CTA

// Twiddle w^n = e^{2 pi i n / M} from the two shared-memory tables of the
// CTA's lattice: w^n = Thi[n >> bl] * Tlo[n & (2^bl - 1)].
__device__ __forceinline__ double2 tw2(const double2* __restrict__ tlo, const double2* __restrict__ thi,
                                       uint32_t n, int bl) {
  return cmul(thi[n >> bl], tlo[n & ((1u << bl) - 1u)]);
}

// One CTA (256 threads) = one 64 x 64 tile (j1, j2) of one unit and one
// slice of the terms; thread tile 4 x 4 complex (j1 = tx + 16 i, j2 = ty + 16 j).
// Operand tiles are double-buffered in shared memory: each stage is generated
// (integer Barrett, two-level table lookups, recurrences) while the other is
// contracted, with one barrier per stage.
// SPLIT: write the unchirped partial sum of this term slice to `part`
// (reduced in slice order by poly_split_reduce_kernel, deterministic).
template <bool SPLIT>
__global__ void __launch_bounds__(SP_T, 2)
sample_poly_kernel(PolyPlan pp, LatTable lt, const double2* __restrict__ cprime,
                   const int32_t* __restrict__ rres, const int32_t* __restrict__ rjs,
                   const double2* __restrict__ tw, const double2* __restrict__ chirp,
                   double2* __restrict__ buf, int64_t ustride, int apply_chirp,
                   double2* __restrict__ part, int64_t pstride) {
  extern __shared__ double2 sm[];
  // two stages of operand tiles: stage b at sm + b * 2 * KC * PT = {A[KC][PT], B[KC][PT]}
  double2* tlo = sm + 4 * KC * PT;   // [2^bl]
  double2* thi = tlo + (1 << pp.bl); // [nhi]
  const int bid = blockIdx.x;
  int lo = 0, hi = pp.nunits - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pp.tile_start[mid] <= bid) lo = mid; else hi = mid - 1;
  }
  const int u = lo;
  const int l = pp.unit_lat[u], it = pp.unit_it[u];
  const int local = bid - pp.tile_start[u];
  const int q = local % pp.ks;
  const int tau = local / pp.ks;
  const int nt1 = pp.nt1[l];
  const int tj1 = tau % nt1, tj2 = tau / nt1;
  const int64_t M = lt.m[l];
  const uint32_t M32 = (uint32_t)M;
  const uint64_t mu = pp.mu[l];
  const int bl = pp.bl;
  const int64_t J1 = pp.J1[l];
  const uint32_t j1_0 = (uint32_t)tj1 * PT, j2_0 = (uint32_t)tj2 * PT;
  const double2* twl = tw + lt.off[l];
  const int s = pp.s;
  const int h_begin = q * pp.kper;
  const int h_end = min(s, h_begin + pp.kper);
  const double2* cp = cprime + (int64_t)it * s;
  const int32_t* rr = rres + (int64_t)l * s;
  const int32_t* rj = rjs + (int64_t)l * s;

  // stage this lattice's two-level twiddle tables
  const int nlo = 1 << bl;
  const int nhi = (int)((M + nlo - 1) >> bl);
  for (int i = threadIdx.x; i < nlo; i += SP_T) tlo[i] = __ldg(&twl[i < M ? i : 0]);
  for (int i = threadIdx.x; i < nhi; i += SP_T) thi[i] = __ldg(&twl[(int64_t)i << bl]);

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = (lane & 7) + 8 * (w & 1);
  const int ty = (lane >> 3) + 4 * (w >> 1);

  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);

  // Operand generation, term-major: the 16 threads of term gh produce rows
  // gt + 16 i of A and B from one table lookup each plus a recurrence by
  // w^{16 r} (3 complex multiplications, a few ulp).
  const int gh = threadIdx.x >> 4, gt = threadIdx.x & 15;
  uint32_t pr = 0, pq = 0;
  double2 pc = make_double2(0.0, 0.0);
  auto fetch = [&](int k0) {
    const int h = k0 + gh;
    if (h < h_end) {
      pr = (uint32_t)__ldg(&rr[h]);
      pq = (uint32_t)__ldg(&rj[h]);
      pc = __ldg(&cp[h]);
    }
  };
  // generation state of the stage being produced
  double2 gv = make_double2(0.0, 0.0), ge = make_double2(1.0, 0.0);
  auto gen_start_a = [&](bool live) {
    gv = make_double2(0.0, 0.0);
    ge = make_double2(1.0, 0.0);
    if (live) {
      gv = cmul(pc, tw2(tlo, thi, mod_barrett((uint64_t)pr * (j1_0 + gt), M32, mu), bl));
      ge = tw2(tlo, thi, mod_barrett((uint64_t)pr * 16u, M32, mu), bl);
    }
  };
  auto gen_start_b = [&](bool live) {
    gv = make_double2(1.0, 0.0);
    ge = make_double2(1.0, 0.0);
    if (live) {
      gv = tw2(tlo, thi, mod_barrett((uint64_t)pq * (j2_0 + gt), M32, mu), bl);
      ge = tw2(tlo, thi, mod_barrett((uint64_t)pq * 16u, M32, mu), bl);
    }
  };
  auto gen_put = [&](double2* dst, int i) {
    dst[gh * PT + gt + 16 * i] = gv;
    if (i < 3) gv = cmul(gv, ge);
  };

  int stage = 0;
  fetch(h_begin);
  __syncthreads();  // tables staged
  if (h_begin < h_end) {
    const bool live = h_begin + gh < h_end;
    gen_start_a(live);
#pragma unroll
    for (int i = 0; i < 4; ++i) gen_put(sm, i);
    gen_start_b(live);
#pragma unroll
    for (int i = 0; i < 4; ++i) gen_put(sm + KC * PT, i);
  }
  fetch(h_begin + KC);
  for (int k0 = h_begin; k0 < h_end; k0 += KC) {
    __syncthreads();  // stage `stage` complete; the other stage is free
    const double2* As = sm + stage * 2 * KC * PT;
    const double2* Bs = As + KC * PT;
    double2* An = sm + (stage ^ 1) * 2 * KC * PT;
    double2* Bn = An + KC * PT;
    const bool more = k0 + KC < h_end;
    const bool live = more && (k0 + KC + gh < h_end);
    if (more) {
      gen_start_a(live);
#pragma unroll
      for (int i = 0; i < 4; ++i) gen_put(An, i);
      gen_start_b(live);
#pragma unroll
      for (int i = 0; i < 4; ++i) gen_put(Bn, i);
      fetch(k0 + 2 * KC);
    }
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      double2 b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk * PT + ty + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 a = As[kk * PT + tx + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fma(a.x, b[j].x, acc[i][j].x);
          acc[i][j].x = fma(-a.y, b[j].y, acc[i][j].x);
          acc[i][j].y = fma(a.x, b[j].y, acc[i][j].y);
          acc[i][j].y = fma(a.y, b[j].x, acc[i][j].y);
        }
      }
    }
    stage ^= 1;
  }
  const double2* ch = chirp + lt.off[l];
  double2* ub = SPLIT ? part + ((int64_t)q * pp.nunits + u) * pstride : buf + (int64_t)u * ustride;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t base = J1 * (int64_t)(j2_0 + ty + 16 * j);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t n = j1_0 + tx + 16 * i + base;
      if (n < M) ub[n] = (!SPLIT && apply_chirp) ? cmul(acc[i][j], __ldg(&ch[n])) : acc[i][j];
    }
  }
}

// sum the term slices of every unit in slice order, then pre-chirp
__global__ void poly_split_reduce_kernel(UnitTable ut, int ks, const double2* __restrict__ part,
                                         int64_t pstride, const double2* __restrict__ chirp,
                                         double2* __restrict__ buf, int64_t ustride, int apply_chirp) {
  const int u = blockIdx.y;
  const int l = ut.lat[u];
  const int64_t M = ut.m[l];
  const double2* ch = chirp + ut.off[l];
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < M;
       n += (int64_t)gridDim.x * blockDim.x) {
    double2 v = part[(int64_t)u * pstride + n];
    for (int q = 1; q < ks; ++q) v = cadd(v, part[((int64_t)q * ut.nunits + u) * pstride + n]);
    buf[(int64_t)u * ustride + n] = apply_chirp ? cmul(v, __ldg(&ch[n])) : v;
  }
}

// ---------------------------------------------------------------------------
// B-spline oracle (testbed.py:198-244): f(x) = sum_g prod_{c in A_g} C_m m B_m(m x_c)

template <bool FAST>
__global__ void sample_bspline_kernel(UnitTable ut, LatTable lt, BsplineSpec bs, AnchorTable at,
                                      const double2* __restrict__ chirp, double2* __restrict__ buf,
                                      int64_t ustride, int apply_chirp) {
  const int u = blockIdx.y;
  const int l = ut.lat[u], it = ut.it[u];
  const int64_t M = lt.m[l];
  const double invM = lt.inv_m[l];
  const int t1 = lt.d;
  const int tail = bs.d - t1;
  const double2* ch = chirp + lt.off[l];
  double2* ub = buf + (int64_t)u * ustride;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < M;
       n += (int64_t)gridDim.x * blockDim.x) {
    double total = 0.0;
    for (int g = 0; g < bs.ngroups; ++g) {
      const int m = bs.order[g];
      double term = 1.0;
      for (int q = bs.start[g]; q < bs.start[g + 1]; ++q) {
        const int c = bs.comps[q];
        double x;
        if (c < t1) {
          const int64_t r = mulmod<FAST>(n, (int64_t)lt.z[l * t1 + c], M, invM);
          x = (double)r * invM;  // within 1 ulp of r / M (the reference's node), no FP64 division
        } else {
          x = at.a[it * tail + (c - t1)];
        }
        term = term * (bs.scale[g] * cardinal_bspline(m, (double)m * x));
      }
      total += term;
    }
    if (apply_chirp) {
      const double2 c = __ldg(&ch[n]);
      ub[n] = make_double2(total * c.x, total * c.y);  // (total + 0i) * c
    } else {
      ub[n] = make_double2(total, 0.0);
    }
  }
}

// in-place x_n <- (x_n + sigma_u (noise_n)) * chirp_n for n < M (host-callback and noisy oracles)
__global__ void finish_samples_kernel(UnitTable ut, const double2* __restrict__ chirp,
                                      double2* __restrict__ buf, int64_t ustride,
                                      const double2* __restrict__ noise, int64_t nstride,
                                      const double* __restrict__ sigma) {
  const int u = blockIdx.y;
  const int l = ut.lat[u];
  const int64_t M = ut.m[l];
  const double2* ch = chirp + ut.off[l];
  double2* ub = buf + (int64_t)u * ustride;
  const double sg = noise ? sigma[u] : 0.0;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < M;
       n += (int64_t)gridDim.x * blockDim.x) {
    double2 v = ub[n];
    if (noise) {
      const double2 e = noise[(int64_t)u * nstride + n];
      v = make_double2(v.x + sg * e.x, v.y + sg * e.y);
    }
    ub[n] = cmul(v, __ldg(&ch[n]));
  }
}

// ---------------------------------------------------------------------------
// Device noise (counter-based, reproducible for any launch split / GPU count):
// Philox4x32-10 keyed by the oracle seed, counter (sample n, oracle-call
// index); Box-Muller gives one complex N(0,1) + i N(0,1) sample per counter.
// The call index is the position of the oracle call in the reference's call
// order (testbed.py:100-106 draws per call), so unit u of a chunk is call
// call_base + (global unit id).

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__device__ __forceinline__ double2 normal2(uint64_t seed, uint64_t call, uint64_t n) {
  uint32_t c[4] = {(uint32_t)n, (uint32_t)(n >> 32), (uint32_t)call, (uint32_t)(call >> 32)};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t a = ((uint64_t)c[0] << 32 | c[1]) >> 11;
  const uint64_t b = ((uint64_t)c[2] << 32 | c[3]) >> 11;
  const double u1 = ((double)a + 1.0) * 0x1.0p-53;  // (0, 1]
  const double u2 = (double)b * 0x1.0p-53;          // [0, 1)
  const double rad = sqrt(-2.0 * log(u1));
  double s, co;
  sincospi(2.0 * u2, &s, &co);
  return make_double2(rad * co, rad * s);
}

// x_n <- (x_n + s_u * (g_re + i g_im)) * chirp_n: s_u = sigma / sqrt(2) (fixed) or
// rel * sqrt(norm2_u / M) / sqrt(2) (relative to the noise-free vector)
__global__ void finish_devnoise_kernel(UnitTable ut, const double2* __restrict__ chirp,
                                       double2* __restrict__ buf, int64_t ustride,
                                       const double* __restrict__ norm2, double rel, double sigma,
                                       uint64_t seed, uint64_t call_base, int apply_chirp) {
  const int u = blockIdx.y;
  const int l = ut.lat[u];
  const int64_t M = ut.m[l];
  const double2* ch = chirp + ut.off[l];
  double2* ub = buf + (int64_t)u * ustride;
  const uint64_t call = call_base + (uint64_t)(ut.it[u] * ut.nlat + l);
  const double sg = (norm2 ? rel * sqrt(norm2[u] / (double)M) : sigma) * 0.70710678118654752440;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < M;
       n += (int64_t)gridDim.x * blockDim.x) {
    const double2 e = normal2(seed, call, (uint64_t)n);
    double2 v = ub[n];
    v = make_double2(v.x + sg * e.x, v.y + sg * e.y);
    ub[n] = apply_chirp ? cmul(v, __ldg(&ch[n])) : v;
  }
}

int launch_finish_devnoise(const UnitTable& ut, const double2* chirp, double2* buf, int64_t ustride,
                           const double* norm2, double rel, double sigma, uint64_t seed,
                           uint64_t call_base, bool apply_chirp, int num_sms, cudaStream_t st) {
  int64_t mmax = 1;
  for (int l = 0; l < ut.nlat; ++l) mmax = ut.m[l] > mmax ? ut.m[l] : mmax;
  int bx = (int)((mmax + 255) / 256);
  const int cap = (num_sms * 8 + ut.nunits - 1) / ut.nunits + 1;
  if (bx > cap) bx = cap;
  finish_devnoise_kernel<<<dim3(bx, ut.nunits), 256, 0, st>>>(ut, chirp, buf, ustride, norm2, rel, sigma,
                                                              seed, call_base, apply_chirp ? 1 : 0);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// squared 2-norm of each unit's first M samples (for relative-noise oracles).
// Deterministic: a cluster of NORM_CL CTAs per unit, each CTA a fixed
// strided slice reduced in a fixed tree, the CTA partials summed in rank
// order by rank 0 through distributed shared memory.  The rounding depends
// on nothing but the unit's samples (not on which units share the launch,
// i.e. not on the GPU count of a sharded step).
constexpr int NORM_CL = 8;
constexpr int NORM_NT = 512;

__global__ void __cluster_dims__(NORM_CL, 1, 1) __launch_bounds__(NORM_NT)
unit_norm2_kernel(UnitTable ut, const double2* __restrict__ buf, int64_t ustride, double* __restrict__ out) {
  __shared__ double red[NORM_NT / 32];
  __shared__ double part;
  const int u = blockIdx.y;
  const int64_t M = ut.m[ut.lat[u]];
  const double2* ub = buf + (int64_t)u * ustride;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  double acc = 0.0;
  for (int64_t n = (int64_t)rank * NORM_NT + threadIdx.x; n < M; n += (int64_t)NORM_CL * NORM_NT) {
    const double2 v = __ldcs(&ub[n]);
    acc = fma(v.x, v.x, fma(v.y, v.y, acc));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < NORM_NT / 32; ++w) t += red[w];
    part = t;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank == 0 && threadIdx.x == 0) {
    double t = 0.0;
    const uint32_t local = (uint32_t)__cvta_generic_to_shared(&part);
    for (uint32_t c = 0; c < NORM_CL; ++c) {
      uint32_t remote;
      double v;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(c));
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
      t += v;
    }
    out[u] = t;
  }
  // no CTA may exit while rank 0 still reads its shared memory
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// B-spline sampler with the lattice work shared by the iterations
// (K1b).  The units of one lattice differ only in the anchor tail, so per node
// the factors of the lattice coordinates are evaluated once, grouped
//   G_g(n) = prod_{c in A_g, c < t1} C_m m B_m(m x_c(n)),
// and unit i gets total_i = sum_g K_{i,g} G_g(n) with the anchor factors
// K_{i,g} = prod_{c in A_g, c >= t1} C_m m B_m(m a_{i,c}) computed once per CTA.
// B_m is evaluated as its piecewise polynomial (Horner in t = u - floor(u),
// bs.pc) instead of the Cox-de Boor triangle.  Grid: (node blocks, lattice).
template <int M_>
__device__ __forceinline__ double bs_horner_t(const double* __restrict__ pc, double u) {
  int iv = (int)u;  // u >= 0
  if (iv > M_ - 1) iv = M_ - 1;
  const double t = u - (double)iv;
  const double* c = pc + bs_poff(M_) + iv * M_;
  double v = c[M_ - 1];
#pragma unroll
  for (int k = M_ - 2; k >= 0; --k) v = fma(v, t, c[k]);
  return v;
}

__device__ __forceinline__ double bs_horner(const double* __restrict__ pc, int m, double u) {
  switch (m) {
    case 1: return u < 1.0 ? 1.0 : 0.0;
    case 2: return bs_horner_t<2>(pc, u);
    case 3: return bs_horner_t<3>(pc, u);
    case 4: return bs_horner_t<4>(pc, u);
    case 5: return bs_horner_t<5>(pc, u);
    case 6: return bs_horner_t<6>(pc, u);
    default: return bs_horner_t<7>(pc, u);
  }
}

constexpr int BS_SLOTS = 8;

template <bool FAST>
__global__ void __launch_bounds__(256)
sample_bspline_lat_kernel(UnitTable ut, LatTable lt, BsplineSpec bs, AnchorTable at,
                          const double2* __restrict__ chirp, double2* __restrict__ buf, int64_t ustride,
                          int apply_chirp) {
  __shared__ double pc[140];
  __shared__ double K[BS_SLOTS][8];
  __shared__ int slot[SFFT_UMAX];
  __shared__ int nslot;
  const int l = blockIdx.y;
  const int t1 = lt.d;
  const int tail = bs.d - t1;
  const int G = bs.ngroups;
  for (int i = threadIdx.x; i < 140; i += blockDim.x) pc[i] = bs.pc[i];
  if (threadIdx.x < 32) {  // the launch's units of this lattice, in slot order
    int cnt = 0;
    for (int b = 0; b < ut.nunits; b += 32) {
      const int j = b + (int)threadIdx.x;
      const bool hit = j < ut.nunits && ut.lat[j] == l;
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (hit) slot[cnt + __popc(bal & ((1u << threadIdx.x) - 1u))] = j;
      cnt += __popc(bal);
    }
    if (threadIdx.x == 0) nslot = cnt;
  }
  __syncthreads();
  const int ns = nslot;
  if (ns == 0) return;
  for (int c0 = 0; c0 < ns; c0 += BS_SLOTS) {
    const int nc = min(BS_SLOTS, ns - c0);
    __syncthreads();
    for (int q = threadIdx.x; q < nc * G; q += blockDim.x) {  // anchor factors of slot, group
      const int sl = q / G, g = q % G;
      const int it = ut.it[slot[c0 + sl]];
      const int m = bs.order[g];
      double k = 1.0;
      for (int e = bs.start[g]; e < bs.start[g + 1]; ++e) {
        const int c = bs.comps[e];
        if (c >= t1) k = k * (bs.scale[g] * bs_horner(pc, m, (double)m * at.a[it * tail + (c - t1)]));
      }
      K[sl][g] = k;
    }
    __syncthreads();
    const int64_t M = lt.m[l];
    const double invM = lt.inv_m[l];
    const double2* ch = chirp + lt.off[l];
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < M;
         n += (int64_t)gridDim.x * blockDim.x) {
      double tot[BS_SLOTS];
#pragma unroll
      for (int s = 0; s < BS_SLOTS; ++s) tot[s] = 0.0;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        if (g < G) {
          const int m = bs.order[g];
          double gg = 1.0;
          for (int e = bs.start[g]; e < bs.start[g + 1]; ++e) {
            const int c = bs.comps[e];
            if (c < t1) {
              const int64_t r = mulmod<FAST>(n, (int64_t)lt.z[l * t1 + c], M, invM);
              const double x = (double)r * invM;  // within 1 ulp of r / M, the reference's node
              gg = gg * (bs.scale[g] * bs_horner(pc, m, (double)m * x));
            }
          }
#pragma unroll
          for (int s = 0; s < BS_SLOTS; ++s)
            if (s < nc) tot[s] += K[s][g] * gg;
        }
      }
      double2 cv = make_double2(1.0, 0.0);
      if (apply_chirp) cv = __ldg(&ch[n]);
#pragma unroll
      for (int s = 0; s < BS_SLOTS; ++s)
        if (s < nc) {
          double2* ub = buf + (int64_t)slot[c0 + s] * ustride;
          __stcs(&ub[n], apply_chirp ? make_double2(tot[s] * cv.x, tot[s] * cv.y) : make_double2(tot[s], 0.0));
        }
    }
  }
}

// K1b main variant: the lattice-shared sampler with the per-coordinate work
// made incremental.  Coordinate c of node n has u = m x = m (n z_c mod M) / M;
// each CTA owns a contiguous node range of one lattice (CTAs dealt to the
// lattices in proportion to M_l) and each thread walks n0, n0 + 256, ...,
// carrying per lattice coordinate Q = m (n z_c mod M) as (piece iv, rem),
// Q = iv M + rem: one step adds m (256 z_c mod M) = Dq M + Dr with integer
// carries, so B_m(u) is the piece iv polynomial at t = rem / M (exact
// rational, one multiply by 1/M) -- no modular product, no float floor per
// node.  Coordinates are laid out group-major ("positions") so that the
// registers of every position have compile-time indices (NP positions at most).
struct BsGrid {
  int ncta;                    // CTAs of the launch
  int start[SFFT_LMAX + 1];    // first CTA of lattice l
};

// x mod M for x < 2^63, M < 2^31 (double quotient, off by at most one)
__device__ __forceinline__ uint64_t mod_u64(uint64_t x, uint64_t M, double invM) {
  int64_t r = (int64_t)x - (int64_t)((uint64_t)__dmul_rn((double)x, invM) * M);
  if (r < 0) r += (int64_t)M;
  if (r >= (int64_t)M) r -= (int64_t)M;
  return (uint64_t)r;
}

template <int NP>
__global__ void __launch_bounds__(256, 3)  // <= 85 registers: 3 CTAs (24 warps) per SM (88 gave 2)
sample_bspline_chain_kernel(UnitTable ut, LatTable lt, BsplineSpec bs, AnchorTable at, BsGrid bg,
                            const double2* __restrict__ chirp, double2* __restrict__ buf, int64_t ustride,
                            int apply_chirp) {
  __shared__ double pcg[8][49];      // group g's piece polynomials of order m_g, scaled by C_m m
  __shared__ double K[BS_SLOTS][8];  // anchor factors per slot and group
  __shared__ double C0[BS_SLOTS];    // groups without lattice coordinates: their constant terms
  __shared__ int slot[SFFT_UMAX];
  __shared__ int nslot, npos;
  __shared__ int pmeta[NP];          // m | group << 4 | (last position of its group) << 8
  __shared__ uint32_t pz[NP], pdq[NP], pdr[NP];
  int l = 0;
  while (l + 1 < lt.nlat && (int)blockIdx.x >= bg.start[l + 1]) ++l;
  const int t1 = lt.d;
  const int tail = bs.d - t1;
  const int G = bs.ngroups;
  const int64_t M = lt.m[l];
  const uint32_t Mu = (uint32_t)M;
  const double invM = lt.inv_m[l];
  // this CTA's node range of lattice l (contiguous, a multiple of 256 wide)
  const int cl = (int)blockIdx.x - bg.start[l], ncl = bg.start[l + 1] - bg.start[l];
  const int64_t span = ((M + ncl - 1) / ncl + 255) / 256 * 256;
  const int64_t nb = (int64_t)cl * span, ne = min(M, nb + span);
  for (int i = threadIdx.x; i < 8 * 49; i += blockDim.x) {
    const int g = i / 49, e = i % 49;
    double v = 0.0;
    if (g < G) {
      const int m = bs.order[g];
      if (e < m * m) v = bs.scale[g] * bs.pc[bs_poff(m) + e];
    }
    pcg[g][e] = v;
  }
  if (threadIdx.x < 32) {  // this lattice's units, in slot order
    int cnt = 0;
    for (int b = 0; b < ut.nunits; b += 32) {
      const int j = b + (int)threadIdx.x;
      const bool hit = j < ut.nunits && ut.lat[j] == l;
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (hit) slot[cnt + __popc(bal & ((1u << threadIdx.x) - 1u))] = j;
      cnt += __popc(bal);
    }
    if (threadIdx.x == 0) {
      nslot = cnt;
      int np = 0;
      for (int g = 0; g < G; ++g) {
        int last = -1;
        for (int e = bs.start[g]; e < bs.start[g + 1]; ++e) {
          const int c = bs.comps[e];
          if (c >= t1 || np >= NP) continue;
          const int m = bs.order[g];
          const uint64_t z = (uint64_t)lt.z[l * t1 + c];
          const uint64_t dl = (256u * z) % (uint64_t)M;  // (256 z) mod M
          const uint64_t md = (uint64_t)m * dl;
          pz[np] = (uint32_t)z;
          pdq[np] = (uint32_t)(md / (uint64_t)M);
          pdr[np] = (uint32_t)(md % (uint64_t)M);
          pmeta[np] = m | (g << 4);
          last = np++;
        }
        if (last >= 0) pmeta[last] |= 1 << 8;
      }
      npos = np;
    }
  }
  __syncthreads();
  const int ns = nslot, np = npos;
  if (ns == 0) return;
  const int64_t n0 = nb + threadIdx.x;
  for (int c0 = 0; c0 < ns; c0 += BS_SLOTS) {
    const int nc = min(BS_SLOTS, ns - c0);
    __syncthreads();
    for (int q = threadIdx.x; q < nc * G; q += blockDim.x) {  // anchor factors
      const int sl = q / G, g = q % G;
      const int it = ut.it[slot[c0 + sl]];
      const int m = bs.order[g];
      double k = 1.0;
      for (int e = bs.start[g]; e < bs.start[g + 1]; ++e) {
        const int c = bs.comps[e];
        if (c >= t1) {
          const double u = (double)m * at.a[it * tail + (c - t1)];
          int iv = (int)u;
          if (iv > m - 1) iv = m - 1;
          const double t = u - (double)iv;
          const double* cf = &pcg[g][iv * m];
          double v = cf[m - 1];
          for (int kk = m - 2; kk >= 0; --kk) v = fma(v, t, cf[kk]);
          k = k * v;
        }
      }
      K[sl][g] = k;
    }
    __syncthreads();
    if (threadIdx.x < nc) {  // groups without lattice coordinates contribute their anchor product
      double c = 0.0;
      for (int g = 0; g < G; ++g) {
        bool has = false;
        for (int e = bs.start[g]; e < bs.start[g + 1]; ++e) has |= bs.comps[e] < t1;
        if (!has) c += K[threadIdx.x][g];
      }
      C0[threadIdx.x] = c;
    }
    __syncthreads();
    if (n0 >= ne) continue;  // no barrier below: every thread meets the next slot chunk's barriers
    uint32_t iv[NP], rem[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      iv[p] = 0u;
      rem[p] = 0u;
      if (p < np) {  // exact start: Q = m (n0 z mod M) = iv M + rem
        const uint64_t r = mod_u64((uint64_t)n0 * pz[p], (uint64_t)M, invM);
        const uint64_t Q = (uint64_t)(pmeta[p] & 15) * r;
        const uint64_t qr = mod_u64(Q, (uint64_t)M, invM);
        iv[p] = (uint32_t)__double2ll_rn((double)(Q - qr) * invM);  // exact: Q - qr = iv M, iv < 8
        rem[p] = (uint32_t)qr;
      }
    }
    const double2* chn = chirp + lt.off[l];
    double2 cv = make_double2(1.0, 0.0);
    if (apply_chirp) cv = __ldg(&chn[n0]);
    for (int64_t n = n0; n < ne; n += 256) {
      // the next node's chirp is requested now (its latency hides behind this node's work)
      double2 cnext = make_double2(1.0, 0.0);
      if (apply_chirp && n + 256 < ne) cnext = __ldg(&chn[n + 256]);
      double tot[BS_SLOTS];
#pragma unroll
      for (int s = 0; s < BS_SLOTS; ++s) tot[s] = s < nc ? C0[s] : 0.0;
      double term = 1.0;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        if (p < np) {
          const int meta = pmeta[p];
          const int m = meta & 15, g = (meta >> 4) & 15;
          const double t = (double)rem[p] * invM;
          const double* cf = &pcg[g][iv[p] * m];
          double v = cf[m - 1];
          for (int kk = m - 2; kk >= 0; --kk) v = fma(v, t, cf[kk]);
          term = term * v;
          if (meta & 256) {
#pragma unroll
            for (int s = 0; s < BS_SLOTS; ++s)
              if (s < nc) tot[s] += K[s][g] * term;
            term = 1.0;
          }
          const uint32_t r2 = rem[p] + pdr[p];
          const uint32_t cy = r2 >= Mu ? 1u : 0u;
          rem[p] = r2 - (cy ? Mu : 0u);
          const uint32_t i2 = iv[p] + pdq[p] + cy;
          iv[p] = i2 >= (uint32_t)m ? i2 - (uint32_t)m : i2;
        }
      }
#pragma unroll
      for (int s = 0; s < BS_SLOTS; ++s)
        if (s < nc) {
          double2* ub = buf + (int64_t)slot[c0 + s] * ustride;
          __stcs(&ub[n], apply_chirp ? make_double2(tot[s] * cv.x, tot[s] * cv.y) : make_double2(tot[s], 0.0));
        }
      cv = cnext;
    }
  }
}

// lattice nodes for a host-callback oracle: pts[n, c] (row-major, d columns)
template <bool FAST>
__global__ void lattice_nodes_kernel(LatTable lt, int l, int d, AnchorTable at, int it,
                                     double* __restrict__ pts) {
  const int64_t M = lt.m[l];
  const double invM = lt.inv_m[l];
  const int t1 = lt.d;
  const int tail = d - t1;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < M;
       n += (int64_t)gridDim.x * blockDim.x) {
    for (int c = 0; c < d; ++c) {
      double x;
      if (c < t1) x = (double)mulmod<FAST>(n, (int64_t)lt.z[l * t1 + c], M, invM) / (double)M;
      else x = at.a[it * tail + (c - t1)];
      pts[n * d + c] = x;
    }
  }
}

// ---------------------------------------------------------------------------
// launchers

int launch_poly_prepare(const int32_t* hf, const double2* coef, int s, int d, const LatTable& lt,
                        const PolyPlan& pp, const AnchorTable& at, double2* cprime, int32_t* rres,
                        int32_t* rj, cudaStream_t st) {
  if (s <= 0) return 0;
  int bx = (s + 255) / 256;
  if (bx > 256) bx = 256;
  poly_rotate_kernel<<<dim3(bx, at.rb), 256, 0, st>>>(hf, coef, s, d, lt.d, at, cprime);
  SFFT_CHECK_LAUNCH();
  poly_residue_kernel<<<dim3(bx, lt.nlat), 256, 0, st>>>(hf, s, lt, pp, rres, rj);
  SFFT_CHECK_LAUNCH();
  return 0;
}

size_t sample_poly_smem(int bl, int64_t mmax) {
  const int64_t nlo = (int64_t)1 << bl;
  const int64_t nhi = (mmax + nlo - 1) / nlo;
  return (size_t)(4 * KC * PT + nlo + nhi) * sizeof(double2);
}

int launch_sample_poly(const PolyPlan& pp, const LatTable& lt, const UnitTable& ut,
                       const double2* cprime, const int32_t* rres, const int32_t* rj,
                       const double2* tw, const double2* chirp, double2* buf, int64_t ustride,
                       bool apply_chirp, double2* scratch, int64_t pstride, int num_sms,
                       cudaStream_t st, bool panels_ready) {
  const int ctas = pp.tile_start[pp.nunits];
  if (ctas <= 0) return 0;
  int64_t mmax = 1;
  for (int l = 0; l < lt.nlat; ++l) mmax = lt.m[l] > mmax ? lt.m[l] : mmax;
  const size_t smem = sample_poly_smem(pp.bl, mmax);
  double2* part = scratch + pp.partial_base;  // [B panels | partial sums]
  if (pp.kind >= 1) {
    unsigned* flags = pp.flag_base > 0 ? (unsigned*)(scratch + pp.flag_base) : nullptr;
    bool reduced = false;
    int rc = launch_sample_poly_ws(pp, lt, cprime, rres, rj, tw, chirp, buf, ustride, apply_chirp,
                                   part, pstride, (double*)scratch, panels_ready, flags, &reduced, st);
    if (rc) return rc;
    if (pp.ks > 1 && !reduced) {
      int bx = (int)((mmax + 255) / 256);
      const int cap = (num_sms * 8 + ut.nunits - 1) / ut.nunits + 1;
      if (bx > cap) bx = cap;
      poly_split_reduce_kernel<<<dim3(bx, ut.nunits), 256, 0, st>>>(ut, pp.ks, part, pstride, chirp,
                                                                    buf, ustride, apply_chirp ? 1 : 0);
      SFFT_CHECK_LAUNCH();
    }
    return 0;
  }
  if (pp.ks > 1) {
    cudaError_t e = set_smem_once((const void*)sample_poly_kernel<true>, smem);
    if (e != cudaSuccess) return (int)e;
    prof_mark(PROF_SAMPLE, true, st);
    sample_poly_kernel<true><<<ctas, SP_T, smem, st>>>(pp, lt, cprime, rres, rj, tw, chirp, buf,
                                                      ustride, apply_chirp ? 1 : 0, part, pstride);
    prof_mark(PROF_SAMPLE, false, st);
    SFFT_CHECK_LAUNCH();
    int bx = (int)((mmax + 255) / 256);
    const int cap = (num_sms * 8 + ut.nunits - 1) / ut.nunits + 1;
    if (bx > cap) bx = cap;
    poly_split_reduce_kernel<<<dim3(bx, ut.nunits), 256, 0, st>>>(ut, pp.ks, part, pstride, chirp,
                                                                  buf, ustride, apply_chirp ? 1 : 0);
    SFFT_CHECK_LAUNCH();
  } else {
    cudaError_t e = set_smem_once((const void*)sample_poly_kernel<false>, smem);
    if (e != cudaSuccess) return (int)e;
    prof_mark(PROF_SAMPLE, true, st);
    sample_poly_kernel<false><<<ctas, SP_T, smem, st>>>(pp, lt, cprime, rres, rj, tw, chirp, buf,
                                                       ustride, apply_chirp ? 1 : 0, nullptr, 0);
    prof_mark(PROF_SAMPLE, false, st);
    SFFT_CHECK_LAUNCH();
  }
  return 0;
}

int launch_sample_bspline(const UnitTable& ut, const LatTable& lt, const BsplineSpec& bs,
                          const AnchorTable& at, const double2* chirp, double2* buf,
                          int64_t ustride, bool fast, bool apply_chirp, int num_sms,
                          cudaStream_t st) {
  int64_t mmax = 1;
  for (int l = 0; l < lt.nlat; ++l) mmax = lt.m[l] > mmax ? lt.m[l] : mmax;
  static const bool legacy = [] {
    const char* e = getenv("SFFT_B200_BSPLINE_KERNEL");
    return e && strcmp(e, "unit") == 0;
  }();
  if (!legacy) {
    // one CTA column per lattice; every CTA serves all units of its lattice
    int bx = (int)((mmax + 255) / 256);
    const int cap = (num_sms * 8 + lt.nlat - 1) / lt.nlat;
    if (bx > cap) bx = cap;
    int npos = 0;
    for (int g = 0; g < bs.ngroups; ++g)
      for (int e = bs.start[g]; e < bs.start[g + 1]; ++e) npos += bs.comps[e] < lt.d;
    prof_mark(PROF_SAMPLE, true, st);
    if (npos <= 16 && bs.ngroups <= 8) {
      // CTAs dealt to the lattices in proportion to their sizes; one wave
      // (resident CTAs per SM: 3 for <= 8 positions, 2 for <= 16, by registers)
      BsGrid bg;
      int64_t tot = 0;
      for (int l = 0; l < lt.nlat; ++l) tot += lt.m[l];
      // one wave: resident CTAs per SM from the occupancy calculator
      const void* fk = npos <= 8 ? (const void*)sample_bspline_chain_kernel<8>
                                 : (const void*)sample_bspline_chain_kernel<16>;
      int per_sm = 2;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fk, 256, 0) != cudaSuccess || per_sm < 1) {
        (void)cudaGetLastError();
        per_sm = 2;
      }
      const int ncta = num_sms * per_sm > lt.nlat ? num_sms * per_sm : lt.nlat;
      int64_t acc = 0;
      for (int l = 0; l < lt.nlat; ++l) {
        bg.start[l] = (int)((acc * (ncta - lt.nlat)) / tot) + l;  // at least one CTA per lattice
        acc += lt.m[l];
      }
      bg.start[lt.nlat] = ncta;
      bg.ncta = ncta;
      if (npos <= 8)
        sample_bspline_chain_kernel<8><<<ncta, 256, 0, st>>>(ut, lt, bs, at, bg, chirp, buf, ustride,
                                                            apply_chirp ? 1 : 0);
      else
        sample_bspline_chain_kernel<16><<<ncta, 256, 0, st>>>(ut, lt, bs, at, bg, chirp, buf, ustride,
                                                             apply_chirp ? 1 : 0);
    } else if (fast)
      sample_bspline_lat_kernel<true><<<dim3(bx, lt.nlat), 256, 0, st>>>(ut, lt, bs, at, chirp, buf, ustride,
                                                                         apply_chirp ? 1 : 0);
    else
      sample_bspline_lat_kernel<false><<<dim3(bx, lt.nlat), 256, 0, st>>>(ut, lt, bs, at, chirp, buf, ustride,
                                                                          apply_chirp ? 1 : 0);
    prof_mark(PROF_SAMPLE, false, st);
    SFFT_CHECK_LAUNCH();
    return 0;
  }
  int bx = (int)((mmax + 255) / 256);
  const int cap = (num_sms * 8 + ut.nunits - 1) / ut.nunits + 1;
  if (bx > cap) bx = cap;
  if (fast)
    sample_bspline_kernel<true><<<dim3(bx, ut.nunits), 256, 0, st>>>(ut, lt, bs, at, chirp, buf,
                                                                     ustride, apply_chirp ? 1 : 0);
  else
    sample_bspline_kernel<false><<<dim3(bx, ut.nunits), 256, 0, st>>>(ut, lt, bs, at, chirp, buf,
                                                                      ustride, apply_chirp ? 1 : 0);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_finish_samples(const UnitTable& ut, const double2* chirp, double2* buf, int64_t ustride,
                          const double2* noise, int64_t nstride, const double* sigma, int num_sms,
                          cudaStream_t st) {
  int64_t mmax = 1;
  for (int l = 0; l < ut.nlat; ++l) mmax = ut.m[l] > mmax ? ut.m[l] : mmax;
  int bx = (int)((mmax + 255) / 256);
  const int cap = (num_sms * 8 + ut.nunits - 1) / ut.nunits + 1;
  if (bx > cap) bx = cap;
  finish_samples_kernel<<<dim3(bx, ut.nunits), 256, 0, st>>>(ut, chirp, buf, ustride, noise,
                                                             nstride, sigma);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_unit_norm2(const UnitTable& ut, const double2* buf, int64_t ustride, double* out,
                      int num_sms, cudaStream_t st) {
  (void)num_sms;
  unit_norm2_kernel<<<dim3(NORM_CL, ut.nunits), NORM_NT, 0, st>>>(ut, buf, ustride, out);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_lattice_nodes(const LatTable& lt, int l, int d, const AnchorTable& at, int it,
                         double* pts, bool fast, cudaStream_t st) {
  int64_t M = lt.m[l];
  int bx = (int)((M + 255) / 256);
  if (bx > 4096) bx = 4096;
  if (fast) lattice_nodes_kernel<true><<<bx, 256, 0, st>>>(lt, l, d, at, it, pts);
  else lattice_nodes_kernel<false><<<bx, 256, 0, st>>>(lt, l, d, at, it, pts);
  SFFT_CHECK_LAUNCH();
  return 0;
}

}  // namespace sfft
