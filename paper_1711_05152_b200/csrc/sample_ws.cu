// K1, warp-specialised variant of the GEMM-factored polynomial sampling
// (see sample.cu for the algebra).  A CTA of 384 threads holds one 64 x 128
// (j1 x j2) output tile: 8 consumer warps contract with 4 x 8 complex register
// tiles per thread (12 shared-memory operand loads per 32 complex MACs, so the
// LSU stays below the DFMA rate), 4 producer warps generate the operand
// stages (Barrett reduction, two-level twiddle tables, short recurrences)
// into a 3-deep ring of shared-memory stages synchronised with named
// barriers (full[s] / empty[s]), so generation overlaps the contraction.
#include "common.cuh"
#include "plan.cuh"
#include "sample.cuh"

namespace sfft {

namespace ws {
constexpr int TJ1 = 64;      // tile rows (j1)
constexpr int TJ2 = 128;     // tile cols (j2)
constexpr int KC = 16;       // terms per stage
constexpr int NS = 3;        // stages
constexpr int NCONS = 256;   // consumer threads (two warpgroups)
constexpr int NPROD = 128;   // producer threads (one warpgroup)
constexpr int REG_CONS = 224;  // setmaxnreg: consumers grow, producers shrink, so that
constexpr int REG_PROD = 56;   // 2 consumer + 1 producer warps fit one SMSP's 16K registers
constexpr int NT = NCONS + NPROD;
constexpr int STAGE = KC * (TJ1 + TJ2);  // complex elements per stage
}  // namespace ws

__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ uint32_t ws_barrett(uint64_t x, uint32_t m, uint64_t mu) {
  const uint64_t q = __umul64hi(x, mu);
  uint64_t r = x - q * (uint64_t)m;
  if (r >= m) r -= m;
  return (uint32_t)r;
}

__device__ __forceinline__ double2 ws_tw(const double2* __restrict__ tlo, const double2* __restrict__ thi,
                                         uint32_t n, int bl) {
  return cmul(thi[n >> bl], tlo[n & ((1u << bl) - 1u)]);
}

template <bool SPLIT>
__global__ void __launch_bounds__(ws::NT, 1)
sample_poly_ws_kernel(PolyPlan pp, LatTable lt, const double2* __restrict__ cprime,
                      const int32_t* __restrict__ rres, const int32_t* __restrict__ rjs,
                      const double2* __restrict__ tw, const double2* __restrict__ chirp,
                      double2* __restrict__ buf, int64_t ustride, int apply_chirp,
                      double2* __restrict__ part, int64_t pstride) {
  using namespace ws;
  extern __shared__ double2 sm[];
  double2* tlo = sm + NS * STAGE;
  double2* thi = tlo + (1 << pp.bl);
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
  const int bl = pp.bl;
  const int64_t J1 = pp.J1[l];
  const uint32_t j1_0 = (uint32_t)tj1 * TJ1, j2_0 = (uint32_t)tj2 * TJ2;
  const double2* twl = tw + lt.off[l];
  const int s = pp.s;
  const int h_begin = q * pp.kper;
  const int h_end = min(s, h_begin + pp.kper);
  const int nchunk = h_end > h_begin ? (h_end - h_begin + KC - 1) / KC : 0;

  const int nlo = 1 << bl;
  const int nhi = (int)((M + nlo - 1) >> bl);
  for (int i = threadIdx.x; i < nlo; i += NT) tlo[i] = __ldg(&twl[i < M ? i : 0]);
  for (int i = threadIdx.x; i < nhi; i += NT) thi[i] = __ldg(&twl[(int64_t)i << bl]);
  __syncthreads();

  if (threadIdx.x >= NCONS) {
    // ---------------- producers ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_PROD));
    const uint32_t M32 = (uint32_t)M;
    const uint64_t mu = pp.mu[l];
    const double2* cp = cprime + (int64_t)it * s;
    const int32_t* rr = rres + (int64_t)l * s;
    const int32_t* rj = rjs + (int64_t)l * s;
    const int pt = threadIdx.x - NCONS;
    const int gh = pt >> 3;  // term of the stage (0..15)
    const int gt = pt & 7;   // row / column phase
    // per-term data prefetched one stage ahead
    uint32_t nr = 0, nq = 0;
    double2 nc = make_double2(0.0, 0.0);
    auto fetch = [&](int c) {
      const int h = h_begin + c * KC + gh;
      if (c < nchunk && h < h_end) {
        nr = (uint32_t)__ldg(&rr[h]);
        nq = (uint32_t)__ldg(&rj[h]);
        nc = __ldg(&cp[h]);
      }
    };
    fetch(0);
    for (int c = 0; c < nchunk; ++c) {
      const int st = c % NS;
      const int h = h_begin + c * KC + gh;
      const bool live = h < h_end;
      const uint32_t r = nr, qq = nq;
      const double2 cf = nc;
      fetch(c + 1);
      if (c >= NS) bar_sync(1 + NS + st, NT);  // consumers released the stage
      double2* As = sm + st * STAGE;
      double2* Bs = As + KC * TJ1;
      // A[gh][gt + 8 i], i < 8: one lookup, recurrence by w^{8 r};
      // B[gh][gt + 8 j], j < 16: lookups at j = 0 and 8, recurrence by w^{8 q}.
      // Three independent chains of 8 per thread.
      double2 ea = make_double2(1.0, 0.0), eb = make_double2(1.0, 0.0);
      double2 v[3];
      v[0] = make_double2(0.0, 0.0);
      v[1] = v[2] = make_double2(1.0, 0.0);
      if (live) {
        ea = ws_tw(tlo, thi, ws_barrett((uint64_t)r * 8u, M32, mu), bl);
        eb = ws_tw(tlo, thi, ws_barrett((uint64_t)qq * 8u, M32, mu), bl);
        v[0] = cmul(cf, ws_tw(tlo, thi, ws_barrett((uint64_t)r * (j1_0 + gt), M32, mu), bl));
        v[1] = ws_tw(tlo, thi, ws_barrett((uint64_t)qq * (j2_0 + gt), M32, mu), bl);
        v[2] = ws_tw(tlo, thi, ws_barrett((uint64_t)qq * (j2_0 + gt + 64u), M32, mu), bl);
      }
      double2* ar = As + gh * TJ1 + gt;
      double2* br = Bs + gh * TJ2 + gt;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        ar[8 * i] = v[0];
        br[8 * i] = v[1];
        br[64 + 8 * i] = v[2];
        if (i < 7) {
          v[0] = cmul(v[0], ea);
          v[1] = cmul(v[1], eb);
          v[2] = cmul(v[2], eb);
        }
      }
      bar_arrive(1 + st, NT);  // stage full
    }
    return;
  }

  // ---------------- consumers ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_CONS));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = lane & 15;               // j1 = tx + 16 i, i < 4
  const int ty = (lane >> 4) + 2 * w;     // j2 = ty + 16 j, j < 8
  double2 acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = make_double2(0.0, 0.0);

  for (int c = 0; c < nchunk; ++c) {
    const int st = c % NS;
    bar_sync(1 + st, NT);  // stage full
    const double2* As = sm + st * STAGE;
    const double2* Bs = As + KC * TJ1;
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      double2 a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk * TJ1 + tx + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[kk * TJ2 + ty + 16 * j];
      // row-major order: 16 consecutive DFMAs share one A component (operand
      // reuse; measured +9% DFMA issue rate over column order, tools/mb_dfma.cu),
      // dependent DFMAs on one accumulator are 16 apart
#pragma unroll
      for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[i][j].x = fma(a[i].x, b[j].x, acc[i][j].x);
          acc[i][j].y = fma(a[i].x, b[j].y, acc[i][j].y);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[i][j].x = fma(-a[i].y, b[j].y, acc[i][j].x);
          acc[i][j].y = fma(a[i].y, b[j].x, acc[i][j].y);
        }
      }
    }
    if (c + NS < nchunk) bar_arrive(1 + NS + st, NT);  // stage empty (only if it will be refilled)
  }
  const double2* ch = chirp + lt.off[l];
  double2* ub = SPLIT ? part + ((int64_t)q * pp.nunits + u) * pstride : buf + (int64_t)u * ustride;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t base = J1 * (int64_t)(j2_0 + ty + 16 * j);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t n = j1_0 + tx + 16 * i + base;
      if (n < M) ub[n] = (!SPLIT && apply_chirp) ? cmul(acc[i][j], __ldg(&ch[n])) : acc[i][j];
    }
  }
}

size_t sample_poly_ws_smem(int bl, int64_t mmax) {
  const int64_t nlo = (int64_t)1 << bl;
  const int64_t nhi = (mmax + nlo - 1) / nlo;
  return (size_t)(ws::NS * ws::STAGE + nlo + nhi) * sizeof(double2);
}

int launch_sample_poly_ws(const PolyPlan& pp, const LatTable& lt, const double2* cprime,
                          const int32_t* rres, const int32_t* rj, const double2* tw,
                          const double2* chirp, double2* buf, int64_t ustride, bool apply_chirp,
                          double2* part, int64_t pstride, cudaStream_t st) {
  const int ctas = pp.tile_start[pp.nunits];
  if (ctas <= 0) return 0;
  int64_t mmax = 1;
  for (int l = 0; l < lt.nlat; ++l) mmax = lt.m[l] > mmax ? lt.m[l] : mmax;
  const size_t smem = sample_poly_ws_smem(pp.bl, mmax);
  const void* fn = pp.ks > 1 ? (const void*)sample_poly_ws_kernel<true> : (const void*)sample_poly_ws_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  prof_mark(PROF_SAMPLE, true, st);
  if (pp.ks > 1)
    sample_poly_ws_kernel<true><<<ctas, ws::NT, smem, st>>>(pp, lt, cprime, rres, rj, tw, chirp, buf,
                                                            ustride, apply_chirp ? 1 : 0, part, pstride);
  else
    sample_poly_ws_kernel<false><<<ctas, ws::NT, smem, st>>>(pp, lt, cprime, rres, rj, tw, chirp, buf,
                                                             ustride, apply_chirp ? 1 : 0, nullptr, 0);
  prof_mark(PROF_SAMPLE, false, st);
  SFFT_CHECK_LAUNCH();
  return 0;
}

}  // namespace sfft
