// K1, warp-specialised variant of the GEMM-factored polynomial sampling
// (see sample.cu for the algebra).  A CTA of 384 threads holds one 64 x 128
// (j1 x j2) output tile: 8 consumer warps contract with 4 x 8 complex register
// tiles per thread (12 shared-memory operand loads per 32 complex MACs, so the
// LSU stays below the DFMA rate), 4 producer warps generate the operand
// stages (Barrett reduction, two-level twiddle tables, short recurrences)
// into a 3-deep ring of shared-memory stages synchronised with named
// barriers (full[s] / empty[s]), so generation overlaps the contraction.
//
// TC = true: the consumers contract on the FP64 tensor cores (DMMA,
// mma.sync m8n8k4 f64: 256 FMAs per warp instruction, measured at 37.1
// TFLOP/s from shared memory on B200 = the DFMA peak, tools/mb_dmma.cu,
// where a DFMA outer product tops out at 84% of it, tools/mb_dfma.cu).  The
// complex product is four real MMAs (Cr += Ar Br - Ai Bi, Ci += Ar Bi + Ai Br)
// and the producers store the operands as split real / imaginary planes in
// MMA fragment order, so every consumer operand load is one conflict-free
// 256 B LDS.64 per warp.  (tcgen05 has no FP64 kind: mma.sync is the FP64
// tensor path on sm_100a.)
#include <cstring>
#include <cstdlib>
#include "common.cuh"
#include "plan.cuh"
#include <atomic>

#include "sample.cuh"

namespace sfft {

namespace ws {
constexpr int TJ1 = 64;      // tile rows (j1)
constexpr int TJ2 = 128;     // tile cols (j2)
constexpr int KC = 16;       // terms per stage
constexpr int NS = 3;        // stages
constexpr int NCONS = 256;   // consumer threads (two warpgroups)
constexpr int NPROD = 128;   // producer threads (one warpgroup)
constexpr int REG_CONS = 224;  // setmaxnreg: consumers grow, producers shrink within the launch's
constexpr int REG_PROD = 56;   // 384 x 168 registers: 256 x (224 - 168) = 128 x (168 - 56).  (232 / 48
                               // would remove the epilogue's 136 B spill but needs 1024 registers more
                               // than the CTA owns: setmaxnreg.inc then waits forever.)
constexpr int NT = NCONS + NPROD;
constexpr int STAGE = KC * (TJ1 + TJ2);  // complex elements per stage
}  // namespace ws

__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// mbarrier handshake (TC path): consumer warps wait on `full` independently
// instead of meeting at a CTA-wide named barrier every stage
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
      ::"r"(smem_addr(b)), "r"(parity) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
// bulk global -> shared copy completing on an mbarrier (no tensor map)
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_addr(b)) : "memory");
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

// D += A B for one 8x8x4 FP64 tile; A (8x4 row) / B (4x8 col) one element per
// lane, D two elements per lane (PTX mma.m8n8k4 fragment layout)
__device__ __forceinline__ void dmma_acc(double2& d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d.x), "+d"(d.y) : "d"(a), "d"(b));
}

template <bool SPLIT, bool TC>
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
  __shared__ uint64_t mbar[2 * NS];  // TC: full[s] (NPROD arrivals), empty[s] (one per consumer warp)
  if (TC && threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&mbar[i], NPROD);
      mbar_init(&mbar[NS + i], NCONS / 32);
    }
  }
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
      if (c >= NS) {  // consumers released the stage
        if (TC) mbar_wait(&mbar[NS + st], ((c / NS) - 1) & 1);
        else bar_sync(1 + NS + st, NT);
      }
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
      if (!TC) {
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
      } else {
        // fragment order: A(j1, h) -> plane[((h>>2) * 8 + (j1>>3)) * 32 + (j1&7) * 4 + (h&3)],
        // B(h, j2) -> plane[((h>>2) * 16 + (j2>>3)) * 32 + (j2&7) * 4 + (h&3)]
        double* a_re = (double*)As;
        double* a_im = a_re + KC * TJ1;
        double* b_re = a_im + KC * TJ1;
        double* b_im = b_re + KC * TJ2;
        const int la = gt * 4 + (gh & 3);
        const int ka = (gh >> 2) * 8 * 32 + la;
        const int kb = (gh >> 2) * 16 * 32 + la;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          a_re[ka + i * 32] = v[0].x;
          a_im[ka + i * 32] = v[0].y;
          b_re[kb + i * 32] = v[1].x;
          b_im[kb + i * 32] = v[1].y;
          b_re[kb + (i + 8) * 32] = v[2].x;
          b_im[kb + (i + 8) * 32] = v[2].y;
          if (i < 7) {
            v[0] = cmul(v[0], ea);
            v[1] = cmul(v[1], eb);
            v[2] = cmul(v[2], eb);
          }
        }
        mbar_arrive(&mbar[st]);  // stage full (release of this thread's stores)
        continue;
      }
      bar_arrive(1 + st, NT);  // stage full
    }
    return;
  }

  // ---------------- consumers ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_CONS));
  if (TC) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int bi0 = (w & 1) * 4;   // 4 row blocks (j1) of 8
    const int bj0 = (w >> 1) * 4;  // 4 column blocks (j2) of 8
    double2 cr[4][4], ci[4][4];    // (.x, .y) = the lane's two columns of the 8x8 block
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) cr[x][y] = ci[x][y] = make_double2(0.0, 0.0);
    for (int c = 0; c < nchunk; ++c) {
      const int st = c % NS;
      mbar_wait(&mbar[st], (c / NS) & 1);  // stage full
      const double* a_re = (const double*)(sm + st * STAGE);
      const double* a_im = a_re + KC * TJ1;
      const double* b_re = a_im + KC * TJ1;
      const double* b_im = b_re + KC * TJ2;
#pragma unroll
      for (int kk = 0; kk < KC / 4; ++kk) {
        double ar[4], ai[4], nai[4], br[4], bm[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          ar[x] = a_re[(kk * 8 + bi0 + x) * 32 + lane];
          ai[x] = a_im[(kk * 8 + bi0 + x) * 32 + lane];
          nai[x] = -ai[x];
        }
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          br[y] = b_re[(kk * 16 + bj0 + y) * 32 + lane];
          bm[y] = b_im[(kk * 16 + bj0 + y) * 32 + lane];
        }
        // four sweeps over the 16 blocks: dependent MMAs on one accumulator are 16 apart
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) dmma_acc(cr[x][y], ar[x], br[y]);
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) dmma_acc(ci[x][y], ar[x], bm[y]);
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) dmma_acc(cr[x][y], nai[x], bm[y]);
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) dmma_acc(ci[x][y], ai[x], br[y]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&mbar[NS + st]);  // stage empty (this warp is done reading it)
    }
    const double2* ch = chirp + lt.off[l];
    double2* ub = SPLIT ? part + ((int64_t)q * pp.nunits + u) * pstride : buf + (int64_t)u * ustride;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int64_t j1 = j1_0 + (bi0 + x) * 8 + (lane >> 2);
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int64_t j2 = j2_0 + (bj0 + y) * 8 + 2 * (lane & 3);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t n = j1 + J1 * (j2 + e);
          const double2 v = make_double2(e ? cr[x][y].y : cr[x][y].x, e ? ci[x][y].y : ci[x][y].x);
          if (n < M) ub[n] = (!SPLIT && apply_chirp) ? cmul(v, __ldg(&ch[n])) : v;
        }
      }
    }
    return;
  }
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

// ---------------------------------------------------------------------------
// Persistent TC variant: one CTA per SM walks a contiguous range of work items
// (item = one (tile, term slice), the CTA of the kernel above).  The stage
// ring and its mbarriers run across item boundaries, so the producers fill
// the next item's first stages (reloading the twiddle tables, which only
// they read, when the lattice changes) while the consumers run the previous
// item's epilogue; no per-CTA launch, table load or pipeline fill per item.
// Per item the terms and phases are those of sample_poly_ws_kernel<SPLIT, true>;
// the complex products use the 3-multiplication form (see the consumers).
struct WsItem {
  int u, l, it, q, nchunk, h_begin, h_end;
  uint32_t j1_0, j2_0;
};

__device__ __forceinline__ WsItem ws_item(const PolyPlan& pp, int w) {
  using namespace ws;
  int lo = 0, hi = pp.nunits - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pp.tile_start[mid] <= w) lo = mid; else hi = mid - 1;
  }
  WsItem x;
  x.u = lo;
  x.l = pp.unit_lat[lo];
  x.it = pp.unit_it[lo];
  const int local = w - pp.tile_start[lo];
  x.q = local % pp.ks;
  const int tau = local / pp.ks;
  const int nt1 = pp.nt1[x.l];
  x.j1_0 = (uint32_t)(tau % nt1) * TJ1;
  x.j2_0 = (uint32_t)(tau / nt1) * TJ2;
  x.h_begin = x.q * pp.kper;
  x.h_end = min(pp.s, x.h_begin + pp.kper);
  x.nchunk = x.h_end > x.h_begin ? (x.h_end - x.h_begin + KC - 1) / KC : 0;
  return x;
}

// TMEM (tensor memory, 512 columns x 128 lanes x 32 bit per SM): warp w of a
// warpgroup reaches lanes 32 (w % 4) .. + 31; .32x32b.x64 moves 64 columns
// of the thread's own lane.  Used as a register extension for the K-split
// running sum (this FP64 kernel issues no tcgen05.mma, TMEM is free).
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
               :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// CTA whose contiguous item range [floor(c I / G), floor((c+1) I / G)) holds item w
__device__ __forceinline__ int ws_cta_of(int w, int items, int grid) {
  return (int)((((int64_t)w + 1) * grid - 1) / items);
}
__device__ __forceinline__ int ws_range_begin(int c, int items, int grid) {
  return (int)(((int64_t)c * items) / grid);
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// B operand panels: block b = (lattice l, slice q, column tile tj2, chunk c)
// holds B[h][j2] = w^{(rJ_h j2) mod M} for the chunk's 16 terms and the
// tile's 128 columns, real / imaginary planes in MMA fragment order (the
// stage layout), dead terms (past the slice) = 1.  B depends only on the
// lattice, so every tile along j1 and every iteration share it; the sampling
// producers then fetch it with one bulk copy per stage instead of
// generating it per CTA.
__global__ void __launch_bounds__(128) poly_bpanel_kernel(PolyPlan pp, LatTable lt, const int32_t* __restrict__ rjs,
                                                          const double2* __restrict__ tw, double* __restrict__ panels) {
  using namespace ws;
  const int b = blockIdx.x;
  int l = 0;
  while (l + 1 < lt.nlat && pp.panel_off[l + 1] <= b) ++l;
  const int idx = b - pp.panel_off[l];
  const int ca = idx % pp.nchunk_total;  // absolute 16-term chunk
  const int tj2 = idx / pp.nchunk_total;
  const int64_t M = lt.m[l];
  const uint32_t M32 = (uint32_t)M;
  const uint64_t mu = pp.mu[l];
  const double2* twl = tw + lt.off[l];
  // warp kk owns terms 4 kk .. 4 kk + 3; lane = (j2 & 7) * 4 + (h & 3), the
  // fragment order, so each store of the 16 column blocks is one contiguous
  // 256 B warp access
  const int kk = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hl = kk * 4 + (lane & 3);
  const int col = lane >> 2;  // j2 = 8 bj + col
  const int h = ca * KC + hl;
  const bool live = h < pp.s;
  double* bre = panels + (int64_t)b * (2 * KC * TJ2);
  double* bim = bre + KC * TJ2;
  double2 v = make_double2(1.0, 0.0), e = make_double2(1.0, 0.0);
  if (live) {
    const uint32_t rq = (uint32_t)__ldg(&rjs[(int64_t)l * pp.s + h]);
    v = __ldg(&twl[ws_barrett((uint64_t)rq * (uint32_t)(tj2 * TJ2 + col), M32, mu)]);
    e = __ldg(&twl[ws_barrett((uint64_t)rq * 8u, M32, mu)]);
  }
  // columns j2 >= J2 = ceil(M / J1) only feed outputs n = j1 + J1 j2 >= M,
  // which are discarded: their panel entries are left unwritten
  const int64_t J2 = (M + pp.J1[l] - 1) / pp.J1[l];
#pragma unroll
  for (int bj = 0; bj < TJ2 / 8; ++bj) {
    const int at = (kk * 16 + bj) * 32 + lane;
    if ((int64_t)tj2 * TJ2 + bj * 8 + col < J2) {
      bre[at] = v.x;
      bim[at] = v.y;
    }
    if (bj + 1 < TJ2 / 8) v = cmul(v, e);
  }
}

// L2 prefetch of what the K-split epilogue of item x will read (the owner's
// running sum, the partials of later CTAs, the chirp), issued a few chunks
// before the epilogue so that its loads hit L2
__device__ __forceinline__ void tcp_prefetch_epilogue(const PolyPlan& pp, const LatTable& lt, const WsItem& x, int w,
                                                   int w0, int w1, int items, int bi0, int bj0, int lane,
                                                   const double2* buf, int64_t ustride, const double2* part,
                                                   int64_t pstride, const double2* chirp, int apply_chirp) {
  const int tb = w - x.q;
  if (tb < w0) return;  // not the owner: plain stores only
  const int qe = min(pp.ks - 1, w1 - 1 - tb);
  const bool last = x.q == qe;
  const bool fin = last || x.q == pp.ks - 1;
  if (!(last && qe < pp.ks - 1) && !(fin && apply_chirp)) return;
  const int64_t M = lt.m[x.l];
  const int64_t J1 = pp.J1[x.l];
  const double2* ch = chirp + lt.off[x.l];
  for (int i = 0; i < 4; ++i) {
    const int64_t j1 = x.j1_0 + (bi0 + i) * 8 + (lane >> 2);
    for (int j = 0; j < 4; ++j)
      for (int e = 0; e < 2; ++e) {
        const int64_t n = j1 + J1 * (x.j2_0 + (bj0 + j) * 8 + 2 * (lane & 3) + e);
        if (n >= M) continue;
        if (fin && apply_chirp) asm volatile("prefetch.global.L2 [%0];" ::"l"(ch + n));
        if (last)
          for (int q2 = qe + 1; q2 < pp.ks; ++q2)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(part + ((int64_t)q2 * pp.nunits + x.u) * pstride + n));
      }
  }
  (void)items;
  (void)buf;
  (void)ustride;
}

template <bool SPLIT>
__global__ void __launch_bounds__(ws::NT, 1)
sample_poly_tcp_kernel(PolyPlan pp, LatTable lt, const double2* __restrict__ cprime,
                       const int32_t* __restrict__ rres, const int32_t* __restrict__ rjs,
                       const double2* __restrict__ tw, const double2* __restrict__ chirp,
                       double2* __restrict__ buf, int64_t ustride, int apply_chirp,
                       double2* __restrict__ part, int64_t pstride, const double* __restrict__ panels,
                       unsigned* __restrict__ flags, unsigned epoch) {
  using namespace ws;
  extern __shared__ double2 sm[];
  __shared__ uint64_t mbar[2 * NS];  // full[s] (NPROD arrivals), empty[s] (one per consumer warp)
  double2* tlo = sm + NS * STAGE;
  double2* thi = tlo + (1 << pp.bl);
  const int items = pp.tile_start[pp.nunits];
  const int w0 = (int)(((int64_t)blockIdx.x * items) / gridDim.x);
  const int w1 = (int)(((int64_t)(blockIdx.x + 1) * items) / gridDim.x);
  const int bl = pp.bl;
  const int s = pp.s;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&mbar[i], NPROD);
      mbar_init(&mbar[NS + i], NCONS / 32);
    }
  }
  __syncthreads();

  if (threadIdx.x >= NCONS) {
    // ---------------- producers ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_PROD));
    const int pt = threadIdx.x - NCONS;
    const int gh = pt >> 3;  // term of the stage (0..15)
    const int gt = pt & 7;   // row / column phase
    const int nlo = 1 << bl;
    const int la = gt * 4 + (gh & 3);
    const int ka = (gh >> 2) * 8 * 32 + la;
    const int kb = (gh >> 2) * 16 * 32 + la;
    int cur_lat = -1;
    int gc = 0;  // stage-ring position over all items of this CTA
    for (int w = w0; w < w1; ++w) {
      const WsItem x = ws_item(pp, w);
      const int64_t M = lt.m[x.l];
      if (x.l != cur_lat) {
        bar_sync(1, NPROD);  // every producer is past its last read of the old tables
        const double2* twl = tw + lt.off[x.l];
        const int nhi = (int)((M + nlo - 1) >> bl);
        for (int i = pt; i < nlo; i += NPROD) tlo[i] = __ldg(&twl[i < M ? i : 0]);
        for (int i = pt; i < nhi; i += NPROD) thi[i] = __ldg(&twl[(int64_t)i << bl]);
        bar_sync(1, NPROD);
        cur_lat = x.l;
      }
      const uint32_t M32 = (uint32_t)M;
      const uint64_t mu = pp.mu[x.l];
      const double2* cp = cprime + (int64_t)x.it * s;
      const int32_t* rr = rres + (int64_t)x.l * s;
      const int32_t* rj = rjs + (int64_t)x.l * s;
      uint32_t nr = 0, nq = 0;
      double2 nc = make_double2(0.0, 0.0);
      {
        const int h = x.h_begin + gh;
        if (x.nchunk > 0 && h < x.h_end) {
          nr = (uint32_t)__ldg(&rr[h]);
          nq = (uint32_t)__ldg(&rj[h]);
          nc = __ldg(&cp[h]);
        }
      }
      for (int c = 0; c < x.nchunk; ++c, ++gc) {
        const int st = gc % NS;
        const int h = x.h_begin + c * KC + gh;
        const bool live = h < x.h_end;
        const uint32_t r = nr, qq = nq;
        const double2 cf = nc;
        {  // per-term data one stage ahead
          const int hn = h + KC;
          if (c + 1 < x.nchunk && hn < x.h_end) {
            nr = (uint32_t)__ldg(&rr[hn]);
            nq = (uint32_t)__ldg(&rj[hn]);
            nc = __ldg(&cp[hn]);
          }
        }
        if (gc >= NS) mbar_wait(&mbar[NS + st], ((gc / NS) - 1) & 1);  // consumers released the stage
        double* a_re = (double*)(sm + st * STAGE);
        double* a_im = a_re + KC * TJ1;
        double* b_re = a_im + KC * TJ1;
        if (pt == 0) {
          // B: the precomputed panel, one bulk copy completing on full[st]
          const int tj2 = (int)(x.j2_0 / TJ2);
          const double* src = panels + ((int64_t)pp.panel_off[x.l] + (int64_t)tj2 * pp.nchunk_total +
                                        x.h_begin / KC + c) * (2 * KC * TJ2);
          mbar_expect_tx(&mbar[st], 2 * KC * TJ2 * 8);
          bulk_g2s(b_re, src, 2 * KC * TJ2 * 8, &mbar[st]);
        }
        // A[gh][gt + 8 i], i < 8: one lookup, recurrence by w^{8 r}
        double2 ea = make_double2(1.0, 0.0);
        double2 va = make_double2(0.0, 0.0);
        if (live) {
          ea = ws_tw(tlo, thi, ws_barrett((uint64_t)r * 8u, M32, mu), bl);
          va = cmul(cf, ws_tw(tlo, thi, ws_barrett((uint64_t)r * (x.j1_0 + gt), M32, mu), bl));
        }
        (void)qq;
        (void)kb;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          a_re[ka + i * 32] = va.x;
          a_im[ka + i * 32] = va.y;
          if (i < 7) va = cmul(va, ea);
        }
        mbar_arrive(&mbar[st]);  // stage full (A stored; B lands via complete_tx)
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  // Complex product in the 3-multiplication form: per term chunk
  //   t1 += Re A Re B,  t2 += Im A Im B,  t3 += (Re A + Im A)(Re B + Im B)
  // and at the end Re = t1 - t2, Im = (t3 - t1) - t2: three real MMAs per
  // complex multiply-accumulate instead of four (the FP64 tensor pipe is the
  // bound).  The plane sums are formed in registers from the staged planes.
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_CONS));
  const int lane = threadIdx.x & 31, wv = threadIdx.x >> 5;
  const int bi0 = (wv & 1) * 4;   // 4 row blocks (j1) of 8
  const int bj0 = (wv >> 1) * 4;  // 4 column blocks (j2) of 8
  // K split reduced in this kernel (SPLIT with publish flags): the running
  // sum of the owned tile lives in TMEM, 128 columns per consumer thread
  const bool fused = SPLIT && flags != nullptr;
  __shared__ uint32_t tmem_slot;
  if (fused) {
    if (wv == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_addr(&tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    bar_sync(2, NCONS);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  int gc = 0;
  for (int w = w0; w < w1; ++w) {
    const WsItem x = ws_item(pp, w);
    double2 t1[4][4], t2[4][4], t3[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) t1[i][j] = t2[i][j] = t3[i][j] = make_double2(0.0, 0.0);
    const int pf_at = x.nchunk > 4 ? x.nchunk - 4 : 0;
    for (int c = 0; c < x.nchunk; ++c, ++gc) {
      const int st = gc % NS;
      if (fused && c == pf_at) tcp_prefetch_epilogue(pp, lt, x, w, w0, w1, items, bi0, bj0, lane, buf, ustride,
                                                     part, pstride, chirp, apply_chirp);
      mbar_wait(&mbar[st], (gc / NS) & 1);  // stage full
      const double* a_re = (const double*)(sm + st * STAGE);
      const double* a_im = a_re + KC * TJ1;
      const double* b_re = a_im + KC * TJ1;
      const double* b_im = b_re + KC * TJ2;
#pragma unroll
      for (int kk = 0; kk < KC / 4; ++kk) {
        double ar[4], ai[4], as[4], br[4], bm[4], bs[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          ar[i] = a_re[(kk * 8 + bi0 + i) * 32 + lane];
          ai[i] = a_im[(kk * 8 + bi0 + i) * 32 + lane];
          as[i] = ar[i] + ai[i];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          br[j] = b_re[(kk * 16 + bj0 + j) * 32 + lane];
          bm[j] = b_im[(kk * 16 + bj0 + j) * 32 + lane];
          bs[j] = br[j] + bm[j];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_acc(t1[i][j], ar[i], br[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_acc(t2[i][j], ai[i], bm[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_acc(t3[i][j], as[i], bs[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&mbar[NS + st]);  // stage empty
    }
    // K split reduced in place (fused): the slices of a tile are consecutive
    // items, so the CTA holding slice 0 ("owner") carries the running sum
    // p_0 + p_1 + ... in TMEM from slice to slice, adds the partials of the
    // slices that fell into the next CTAs' ranges (published with a release
    // flag) and writes the chirped total.  The summation order
    // ((p_0 + p_1) + p_2) + ... is that of poly_split_reduce_kernel, so the
    // result is bit-identical to the partials + reduce path (flags == null).
    const int tb = w - x.q;                          // item of the tile's slice 0
    const bool owns = !SPLIT || (fused && tb >= w0);
    const int qe = min(pp.ks - 1, w1 - 1 - tb);      // last slice of the tile in this CTA
    const bool last = !SPLIT || x.q == qe;
    const bool pulls = SPLIT && owns && last && qe < pp.ks - 1;
    if (pulls) {
      const int clast = ws_cta_of(tb + pp.ks - 1, items, gridDim.x);
      for (int c2 = blockIdx.x + 1; c2 <= clast; ++c2) {
        if (ws_range_begin(c2, items, gridDim.x) == ws_range_begin(c2 + 1, items, gridDim.x)) continue;
        while (ld_acquire_u32(&flags[c2]) != epoch) __nanosleep(64);
      }
    }
    // this thread's TMEM columns (re-read here: no register held across the loop)
    const uint32_t taddr = fused ? *(volatile uint32_t*)&tmem_slot + ((uint32_t)(32 * (wv & 3)) << 16) +
                                       (uint32_t)((wv >> 2) * 128)
                                 : 0u;
    // this slice's values (t1..t3 die here): index k = (i * 4 + j) * 2 + e
    double vr[32], vi[32];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double p1 = e ? t1[i][j].y : t1[i][j].x;
          const double p2 = e ? t2[i][j].y : t2[i][j].x;
          const double p3 = e ? t3[i][j].y : t3[i][j].x;
          vr[(i * 4 + j) * 2 + e] = p1 - p2;
          vi[(i * 4 + j) * 2 + e] = (p3 - p1) - p2;
        }
    if (SPLIT && owns && x.q > 0) {
      // S_q = S_{q-1} + p_q, S_{q-1} from TMEM in 4 pieces of 16 values
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        uint32_t r[16];
        tmem_ld16(taddr + h * 16, r);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double pv = __hiloint2double((int)r[2 * k + 1], (int)r[2 * k]);
          if (h < 4) vr[h * 8 + k] = pv + vr[h * 8 + k];
          else vi[(h - 4) * 8 + k] = pv + vi[(h - 4) * 8 + k];
        }
      }
    }
    const int64_t M = lt.m[x.l];
    const int64_t J1 = pp.J1[x.l];
    const double2* ch = chirp + lt.off[x.l];
    double2* bu = buf + (int64_t)x.u * ustride;
    if (pulls) {
      for (int q2 = qe + 1; q2 < pp.ks; ++q2) {
        const double2* src = part + ((int64_t)q2 * pp.nunits + x.u) * pstride;
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 8) {  // 8 loads in flight (registers)
          double2 pv[8];
#pragma unroll
          for (int k = k0; k < k0 + 8; ++k) {
            const int i = k >> 3, j = (k >> 1) & 3, e = k & 1;
            const int64_t n =
                x.j1_0 + (bi0 + i) * 8 + (lane >> 2) + J1 * (x.j2_0 + (bj0 + j) * 8 + 2 * (lane & 3) + e);
            pv[k - k0] = n < M ? __ldcg(&src[n]) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int k = k0; k < k0 + 8; ++k) {
            vr[k] = vr[k] + pv[k - k0].x;
            vi[k] = vi[k] + pv[k - k0].y;
          }
        }
      }
    }
    const bool final_out = owns && (last || x.q == pp.ks - 1);
    if (SPLIT && owns && !final_out) {
      // running sum to TMEM: columns [0, 64) real parts, [64, 128) imaginary
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        uint32_t r[16];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double v = h < 4 ? vr[h * 8 + k] : vi[(h - 4) * 8 + k];
          r[2 * k] = (uint32_t)__double2loint(v);
          r[2 * k + 1] = (uint32_t)__double2hiint(v);
        }
        tmem_st16(taddr + h * 16, r);
      }
      tmem_wait_st();
    } else {
      double2* dst = owns ? bu : part + ((int64_t)x.q * pp.nunits + x.u) * pstride;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int i = k >> 3, j = (k >> 1) & 3, e = k & 1;
        const int64_t n = x.j1_0 + (bi0 + i) * 8 + (lane >> 2) + J1 * (x.j2_0 + (bj0 + j) * 8 + 2 * (lane & 3) + e);
        if (n < M) {
          const double2 v = make_double2(vr[k], vi[k]);
          dst[n] = (final_out && apply_chirp) ? cmul(v, __ldg(&ch[n])) : v;
        }
      }
    }
    if (fused && !owns && last) {
      // this CTA's slices of the tile it entered mid-way are stored: publish
      bar_sync(2, NCONS);
      if (threadIdx.x == 0) {
        __threadfence();
        st_release_u32(&flags[blockIdx.x], epoch);
      }
    }
  }
  if (fused) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    bar_sync(2, NCONS);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (wv == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_slot) : "memory");
  }
}

size_t sample_poly_ws_smem(int bl, int64_t mmax) {
  const int64_t nlo = (int64_t)1 << bl;
  const int64_t nhi = (mmax + nlo - 1) / nlo;
  return (size_t)(ws::NS * ws::STAGE + nlo + nhi) * sizeof(double2);
}

int launch_bpanels(const PolyPlan& pp, const LatTable& lt, const int32_t* rj, const double2* tw, double* panels,
                   cudaStream_t st) {
  if (pp.kind != 2 || pp.npanels <= 0) return 0;
  poly_bpanel_kernel<<<pp.npanels, 128, 0, st>>>(pp, lt, rj, tw, panels);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_sample_poly_ws(const PolyPlan& pp, const LatTable& lt, const double2* cprime,
                          const int32_t* rres, const int32_t* rj, const double2* tw,
                          const double2* chirp, double2* buf, int64_t ustride, bool apply_chirp,
                          double2* part, int64_t pstride, double* panels, bool panels_ready,
                          unsigned* flags, bool* reduced, cudaStream_t st) {
  *reduced = false;
  const int ctas = pp.tile_start[pp.nunits];
  if (ctas <= 0) return 0;
  int64_t mmax = 1;
  for (int l = 0; l < lt.nlat; ++l) mmax = lt.m[l] > mmax ? lt.m[l] : mmax;
  const size_t smem = sample_poly_ws_smem(pp.bl, mmax);
  const bool tc = pp.kind == 2;
  static const bool persistent = [] {
    const char* e = getenv("SFFT_B200_TC_PERSISTENT");
    return !(e && strcmp(e, "0") == 0);
  }();
  static const bool fused = [] {
    const char* e = getenv("SFFT_B200_TC_FUSED_REDUCE");
    return !(e && strcmp(e, "0") == 0);
  }();
  if (!fused) flags = nullptr;
  if (tc && persistent && pp.npanels > 0) {
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int grid = ctas < nsm ? ctas : nsm;
    if (grid > SFFT_WS_MAX_FLAGS) grid = SFFT_WS_MAX_FLAGS;
    const void* fp = pp.ks > 1 ? (const void*)sample_poly_tcp_kernel<true> : (const void*)sample_poly_tcp_kernel<false>;
    cudaError_t e2 = set_smem_once(fp, smem);
    if (e2 != cudaSuccess) return (int)e2;
    // The in-kernel K-split reduction spins on flags published by other CTAs
    // of the grid, so it needs all CTAs co-resident: a cooperative launch
    // (the driver refuses one that cannot be co-resident, e.g. under MPS
    // limits or SMs held by other work) and the flags zeroed on the stream.
    // Without co-residency the slices go through partials + the ordered
    // reduce kernel instead (same rounding: the caller sees *reduced = false).
    if (flags != nullptr && pp.ks > 1) {
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fp, ws::NT, smem) != cudaSuccess ||
          per_sm * nsm < grid)
        flags = nullptr;
    }
    const unsigned epoch = 1u;
    prof_mark(PROF_SAMPLE, true, st);
    if (!panels_ready) poly_bpanel_kernel<<<pp.npanels, 128, 0, st>>>(pp, lt, rj, tw, panels);
    int launched = panels_ready ? 0 : 1;
    if (pp.ks > 1 && flags != nullptr) {
      cudaError_t em = cudaMemsetAsync(flags, 0, sizeof(unsigned) * (size_t)grid, st);
      if (em != cudaSuccess) return (int)em;
      int apply = apply_chirp ? 1 : 0;
      int64_t ustride_ = ustride, pstride_ = pstride;
      unsigned epoch_ = epoch;
      PolyPlan pp_ = pp;
      LatTable lt_ = lt;
      void* args[] = {(void*)&pp_, (void*)&lt_, (void*)&cprime, (void*)&rres, (void*)&rj, (void*)&tw,
                      (void*)&chirp, (void*)&buf, (void*)&ustride_, (void*)&apply, (void*)&part,
                      (void*)&pstride_, (void*)&panels, (void*)&flags, (void*)&epoch_};
      cudaError_t ec = cudaLaunchCooperativeKernel(fp, dim3(grid), dim3(ws::NT), args, smem, st);
      if (ec == cudaErrorCooperativeLaunchTooLarge) {
        (void)cudaGetLastError();
        flags = nullptr;
      } else if (ec != cudaSuccess) {
        return (int)ec;
      } else {
        ++launched;
      }
    }
    if (pp.ks > 1 && flags == nullptr) {
      sample_poly_tcp_kernel<true><<<grid, ws::NT, smem, st>>>(pp, lt, cprime, rres, rj, tw, chirp, buf, ustride,
                                                               apply_chirp ? 1 : 0, part, pstride, panels,
                                                               nullptr, 0u);
      ++launched;
    } else if (pp.ks <= 1) {
      sample_poly_tcp_kernel<false><<<grid, ws::NT, smem, st>>>(pp, lt, cprime, rres, rj, tw, chirp, buf, ustride,
                                                                apply_chirp ? 1 : 0, nullptr, 0, panels,
                                                                nullptr, 0u);
      ++launched;
    }
    prof_mark(PROF_SAMPLE, false, st);
    *reduced = pp.ks == 1 || flags != nullptr;
    SFFT_CHECK_LAUNCHES(launched);
    return 0;
  }
  const void* fn = pp.ks > 1 ? (tc ? (const void*)sample_poly_ws_kernel<true, true>
                                   : (const void*)sample_poly_ws_kernel<true, false>)
                             : (tc ? (const void*)sample_poly_ws_kernel<false, true>
                                   : (const void*)sample_poly_ws_kernel<false, false>);
  cudaError_t e = set_smem_once(fn, smem);
  if (e != cudaSuccess) return (int)e;
  prof_mark(PROF_SAMPLE, true, st);
#define SFFT_WS_LAUNCH(SPLIT, TCV)                                                                      \
  sample_poly_ws_kernel<SPLIT, TCV><<<ctas, ws::NT, smem, st>>>(pp, lt, cprime, rres, rj, tw, chirp, buf, \
                                                                ustride, apply_chirp ? 1 : 0,            \
                                                                SPLIT ? part : nullptr, SPLIT ? pstride : 0)
  if (pp.ks > 1) {
    if (tc) SFFT_WS_LAUNCH(true, true); else SFFT_WS_LAUNCH(true, false);
  } else {
    if (tc) SFFT_WS_LAUNCH(false, true); else SFFT_WS_LAUNCH(false, false);
  }
#undef SFFT_WS_LAUNCH
  prof_mark(PROF_SAMPLE, false, st);
  SFFT_CHECK_LAUNCH();
  return 0;
}

}  // namespace sfft
