// K3: alias histogram, alias-free masks and coverage of one randomized MR1L
// attempt over all L_max pre-drawn lattices at once.
//
// Reference: construct.py:139-143 (_alias_free_mask: residues, bincount,
// counts[res] == 1), construct.py:173-181 (per-prime loop, covered |= mask,
// early exit when covered.all()), lattice.py:511-517 (residues).
//
// Pre-drawing all L_max generating vectors of an attempt is stream-identical
// to the reference's sequential draw (the attempt's generator is discarded
// afterwards, SURVEY §7 hard part 1), so the early exit becomes a reduction:
// candidate k is first covered by lattice ctz(mask_k); the attempt uses
// L = max_k (ctz(mask_k) + 1) lattices when every mask is nonzero.
//
// The histogram only needs "seen once" / "seen at least twice" per bin, so it
// is kept as two bitmaps per lattice (2 bits per residue bin instead of an
// int64 count): seen1 |= bit; if the bit was already set, seen2 |= bit.  The
// result is exact for any multiplicity and the bitmaps (sum_l M_l / 4 bytes)
// stay L2-resident even at |J| = 6.5e5, d = 20 (29 lattices, ~9 MB).
//
// Cluster path (alias_cluster_kernel, opt-in: SFFT_B200_ALIAS_CLUSTER=1; at
// config 1 it measured 60 us against the L2-atomic kernels' 43 us, the
// per-cluster re-reads of J and the DSMEM fold outweigh the atomics saved),
// when a lattice's two bitmaps fit in a CTA's shared memory (M up to ~880k):
// no global atomics.  A thread-block
// cluster (16 CTAs where the GPU allows, else 8) owns a group of lattices;
// each CTA takes a contiguous slice of the candidates and builds the full
// 2-bit histograms of its slice with shared-memory atomics (A); the cluster
// then folds the 16 partial histograms through distributed shared memory,
// each CTA one range of words (B: seen2 |= s2_c | (seen1 & s1_c), seen1 |=
// s1_c, 16-byte DSMEM loads), copies the folded seen2 of every range back
// from its owner (C) and reads each candidate's alias-free bit locally (D),
// writing one bit-plane word per warp and lattice.  alias_planes_kernel then
// folds the planes into the per-candidate 64-bit masks and the stats.
// The default, and larger lattices (config 3, M ~ 1.3e6): the L2-atomic
// kernels below.
#include "common.cuh"
#include "plan.cuh"

#include <cstdlib>
#include <cstring>

namespace sfft {

constexpr int AB = 8;  // lattices per group of independent memory operations

// bitmap word offsets: lattice l owns words [bw[l], bw[l+1]) in each bitmap
__device__ __forceinline__ int64_t bm_words(int64_t m) { return (m + 31) >> 5; }

template <int DM, bool FAST>
__global__ void __launch_bounds__(256)
alias_mark_kernel(const int32_t* __restrict__ freqs, int64_t n, LatTable lt, int l0,
                  uint32_t* __restrict__ seen1, uint32_t* __restrict__ seen2, int64_t words_total) {
  __shared__ int64_t bw[SFFT_LMAX + 1];
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int l = 0; l < lt.nlat; ++l) { bw[l] = acc; acc += bm_words(lt.m[l]); }
    bw[lt.nlat] = acc;
  }
  __syncthreads();
  const int d = lt.d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t k[DM];
    load_cand<DM>(k, freqs, n, i, d);
    // groups of AB lattices: the group's first-bitmap atomics are issued back
    // to back (independent), then the rare second-bitmap ones
    for (int lb = l0; lb < lt.nlat; lb += AB) {
      int64_t w[AB];
      uint32_t bit[AB], old[AB];
#pragma unroll
      for (int j = 0; j < AB; ++j) {
        const int l = lb + j;
        old[j] = 0;
        bit[j] = 0;
        if (l < lt.nlat) {
          const int64_t r = SFFT_RES(DM, FAST, k, lt, l);
          w[j] = bw[l] + (r >> 5);
          bit[j] = 1u << (r & 31);
          old[j] = atomicOr(&seen1[w[j]], bit[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < AB; ++j)
        if (old[j] & bit[j]) atomicOr(&seen2[w[j]], bit[j]);
    }
  }
}

// stats[0] = max_k first-cover index (1-based), stats[1] = #candidates with an empty mask.
// Lattices [l0, nlat): l0 > 0 adds their bits to masks of lattices [0, l0)
// computed by an earlier launch (the stats then cover all nlat lattices).
template <int DM, bool FAST>
__global__ void __launch_bounds__(256)
alias_mask_kernel(const int32_t* __restrict__ freqs, int64_t n, LatTable lt, int l0,
                  const uint32_t* __restrict__ seen2, uint64_t* __restrict__ masks,
                  int32_t* __restrict__ stats) {
  __shared__ int64_t bw[SFFT_LMAX + 1];
  __shared__ int red[32];
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int l = 0; l < lt.nlat; ++l) { bw[l] = acc; acc += bm_words(lt.m[l]); }
    bw[lt.nlat] = acc;
  }
  __syncthreads();
  const int d = lt.d;
  int first_max = 0, empty = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t k[DM];
    load_cand<DM>(k, freqs, n, i, d);
    uint64_t mask = l0 > 0 ? masks[i] : 0ull;
    for (int lb = l0; lb < lt.nlat; lb += AB) {
      uint32_t wv[AB];
      int sh[AB];
#pragma unroll
      for (int j = 0; j < AB; ++j) {  // the group's loads in flight together
        const int l = lb + j;
        wv[j] = ~0u;
        sh[j] = 0;
        if (l < lt.nlat) {
          const int64_t r = SFFT_RES(DM, FAST, k, lt, l);
          sh[j] = (int)(r & 31);
          wv[j] = __ldg(&seen2[bw[l] + (r >> 5)]);
        }
      }
#pragma unroll
      for (int j = 0; j < AB; ++j)
        if (!((wv[j] >> sh[j]) & 1u)) mask |= (1ull << (lb + j));
    }
    masks[i] = mask;
    if (mask) first_max = max(first_max, __ffsll((long long)mask));
    else empty += 1;
  }
  // block reductions
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    first_max = max(first_max, __shfl_down_sync(0xffffffffu, first_max, o));
    empty += __shfl_down_sync(0xffffffffu, empty, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { red[wid] = first_max; red[16 + wid] = empty; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int fm = 0, em = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { fm = max(fm, red[w]); em += red[16 + w]; }
    if (fm) atomicMax(&stats[0], fm);
    if (em) atomicAdd(&stats[1], em);
  }
}

// ---------------------------------------------------------------------------
// cluster / DSMEM variant

struct AliasGroups {
  int l0;      // first lattice of the launch
  int nl;      // lattices of the launch
  int g;       // lattices per cluster
  int wpc;     // bitmap words per CTA and bitmap
  int keep;    // residues of pass 1 kept in shared memory for pass 2
  int64_t sl;  // candidates per CTA slice (multiple of 32)
};

__device__ __forceinline__ uint32_t dsm_map(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int ACT = 1024;  // threads per CTA (one CTA per SM; latency hiding by width)

template <int DM, bool FAST>
__global__ void __launch_bounds__(ACT)
alias_cluster_kernel(const int32_t* __restrict__ freqs, int64_t n, LatTable lt, AliasGroups ag,
                     uint32_t* __restrict__ planes, int64_t pwords) {
  // [g][seen1 | seen2][W] full bitmaps of this CTA's candidates, then (keep) residues [g][sl]
  extern __shared__ uint32_t bm[];
  uint32_t rank, nct;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nct));
  const int cid = (int)(blockIdx.x / nct);
  const int lb = ag.l0 + cid * ag.g;
  const int le = min(ag.l0 + ag.nl, lb + ag.g);
  const int ng = le - lb;
  const int W = ag.wpc;  // words per bitmap (multiple of 4 * cluster size)
  uint32_t* res_s = bm + 2 * ag.g * W;
  for (int w = threadIdx.x; w < ng * 2 * W; w += blockDim.x) bm[w] = 0u;
  __syncthreads();
  const int64_t i0 = min(n, (int64_t)rank * ag.sl);
  const int64_t i1 = min(n, i0 + ag.sl);
  const int d = lt.d;
  // A: local 2-bit saturating histograms of this CTA's candidates
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    int32_t k[DM];
    load_cand<DM>(k, freqs, n, i, d);
    for (int j = 0; j < ng; ++j) {
      const uint32_t r = (uint32_t)SFFT_RES(DM, FAST, k, lt, lb + j);
      if (ag.keep) res_s[(int64_t)j * ag.sl + (i - i0)] = r;
      uint32_t* s1 = bm + 2 * j * W;
      const uint32_t bit = 1u << (r & 31);
      const uint32_t old = atomicOr(&s1[r >> 5], bit);
      if (old & bit) atomicOr(&s1[W + (r >> 5)], bit);
    }
  }
  cluster_barrier();
  // B: fold the cluster's histograms on this CTA's quarter-words
  // (seen2 |= s2_c | (seen1 & s1_c); seen1 |= s1_c), result into local seen2
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(bm);
  const int q4 = W / 4 / (int)nct;  // uint4 words per CTA and bitmap
  for (int x = threadIdx.x; x < ng * q4; x += blockDim.x) {
    const int j = x / q4;
    const int w4 = (int)rank * q4 + x % q4;
    const uint32_t o1 = 4u * (uint32_t)(2 * j * W + 4 * w4), o2 = o1 + 4u * (uint32_t)W;
    uint4 a1 = make_uint4(0, 0, 0, 0), a2 = make_uint4(0, 0, 0, 0);
    for (uint32_t c = 0; c < nct; ++c) {
      uint4 x1, x2;
      asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(x1.x), "=r"(x1.y), "=r"(x1.z), "=r"(x1.w) : "r"(dsm_map(base + o1, c)) : "memory");
      asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(x2.x), "=r"(x2.y), "=r"(x2.z), "=r"(x2.w) : "r"(dsm_map(base + o2, c)) : "memory");
      a2.x |= x2.x | (a1.x & x1.x); a2.y |= x2.y | (a1.y & x1.y);
      a2.z |= x2.z | (a1.z & x1.z); a2.w |= x2.w | (a1.w & x1.w);
      a1.x |= x1.x; a1.y |= x1.y; a1.z |= x1.z; a1.w |= x1.w;
    }
    *(uint4*)(bm + 2 * j * W + W + 4 * w4) = a2;  // only this CTA reads this range of its seen2
  }
  cluster_barrier();
  // C: the folded seen2 of every range, from its owner, into local seen1
  for (int x = threadIdx.x; x < ng * (W / 4); x += blockDim.x) {
    const int j = x / (W / 4);
    const int w4 = x % (W / 4);
    const uint32_t owner = (uint32_t)(w4 / q4);
    uint4 v;
    asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(dsm_map(base + 4u * (uint32_t)(2 * j * W + W + 4 * w4), owner)) : "memory");
    *(uint4*)(bm + 2 * j * W + 4 * w4) = v;
  }
  __syncthreads();
  // D: alias-free bits (final seen2 clear), one bit-plane word per warp and lattice
  const int lane = threadIdx.x & 31;
  for (int64_t ib = i0; ib < i1; ib += blockDim.x) {
    const int64_t i = ib + threadIdx.x;
    const bool live = i < i1;
    int32_t k[DM];
    if (!ag.keep) {
      load_cand<DM>(k, freqs, n, i, d, live);
    }
    for (int j = 0; j < ng; ++j) {
      uint32_t free = 0u;
      if (live) {
        const uint32_t r = ag.keep ? res_s[(int64_t)j * ag.sl + (i - i0)]
                                   : (uint32_t)SFFT_RES(DM, FAST, k, lt, lb + j);
        free = ((bm[2 * j * W + (r >> 5)] >> (r & 31)) & 1u) ? 0u : 1u;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, free);
      if (lane == 0 && ib + (threadIdx.x & ~31) < i1)
        planes[(int64_t)(lb + j - ag.l0) * pwords + ((ib + threadIdx.x) >> 5)] = bal;
    }
  }
  cluster_barrier();  // no CTA leaves while others may still read its seen2
}

// alias-free bit-planes of lattices [l0, l1) -> masks (OR-ed into the masks of
// [0, l0) when l0 > 0), stats as alias_mask_kernel
__global__ void __launch_bounds__(256)
alias_planes_kernel(int64_t n, int l0, int l1, const uint32_t* __restrict__ planes, int64_t pwords,
                    uint64_t* __restrict__ masks, int32_t* __restrict__ stats) {
  __shared__ int red[32];
  int first_max = 0, empty = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t mask = l0 > 0 ? masks[i] : 0ull;
    for (int l = l0; l < l1; ++l)
      mask |= (uint64_t)((__ldg(&planes[(int64_t)(l - l0) * pwords + (i >> 5)]) >> (i & 31)) & 1u) << l;
    masks[i] = mask;
    if (mask) first_max = max(first_max, __ffsll((long long)mask));
    else empty += 1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    first_max = max(first_max, __shfl_down_sync(0xffffffffu, first_max, o));
    empty += __shfl_down_sync(0xffffffffu, empty, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { red[wid] = first_max; red[16 + wid] = empty; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int fm = 0, em = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { fm = max(fm, red[w]); em += red[16 + w]; }
    if (fm) atomicMax(&stats[0], fm);
    if (em) atomicAdd(&stats[1], em);
  }
}

namespace {
constexpr size_t ALIAS_SMEM_MAX = 220 * 1024;

// Cluster geometry for lattices [l0, l1): the largest cluster (16 CTAs where
// allowed, else 8) and the fewest lattices per cluster g such that the
// clusters are resident at once (one wave, one CTA per SM) and a group's
// bitmaps fit in its shared memory; residues are kept for pass 2 when they
// fit too.  False when no geometry fits (the L2-atomic kernels then run).
template <int DM, bool FAST>
bool alias_cluster_plan(const LatTable& lt, int64_t n, int l0, int l1, int& cl, AliasGroups& ag, int& clusters,
                        size_t& smem) {
  // opt-in (SFFT_B200_ALIAS_CLUSTER=1): measured 60 us against the L2-atomic
  // kernels' 43 us at config 1 (tools/alias_ab.py, profiles/r02_alias_ab.jsonl)
  static const bool disabled = [] {
    const char* e = getenv("SFFT_B200_ALIAS_CLUSTER");
    return !(e && strcmp(e, "1") == 0);
  }();
  if (disabled) return false;
  int64_t mw = 1;
  for (int l = l0; l < l1; ++l) mw = max(mw, (lt.m[l] + 31) >> 5);
  const void* fn = (const void*)alias_cluster_kernel<DM, FAST>;
  const int nl = l1 - l0;
  for (int c : {16, 8}) {
    const int wpc = (int)((mw + 4 * c - 1) / (4 * c)) * 4 * c;  // full bitmap words, a multiple of 4 c
    const size_t per_lat = (size_t)2 * wpc * 4;
    if (per_lat > ALIAS_SMEM_MAX) continue;
    if (c > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      (void)cudaGetLastError();
      continue;
    }
    const int64_t sl = (((n + 31) / 32 + c - 1) / c) * 32;
    for (int g = 1; g <= nl; ++g) {
      const int need = (nl + g - 1) / g;
      size_t sm = per_lat * g;
      if (sm > ALIAS_SMEM_MAX) break;
      const size_t with_res = sm + (size_t)g * sl * 4;
      const bool keep = with_res <= ALIAS_SMEM_MAX;
      if (keep) sm = with_res;
      if (set_smem_once(fn, sm) != cudaSuccess) { (void)cudaGetLastError(); break; }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c, 1, 1);
      cfg.blockDim = dim3(ACT, 1, 1);
      cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int maxc = 0;
      if (cudaOccupancyMaxActiveClusters(&maxc, fn, &cfg) != cudaSuccess) { (void)cudaGetLastError(); break; }
      if (maxc >= need) {
        cl = c;
        ag.l0 = l0;
        ag.nl = nl;
        ag.g = g;
        ag.wpc = wpc;
        ag.keep = keep ? 1 : 0;
        ag.sl = sl;
        clusters = need;
        smem = sm;
        return true;
      }
    }
  }
  return false;
}
}  // namespace

template <int DM, bool FAST>
static int launch_alias_cluster_t(const int32_t* freqs, int64_t n, const LatTable& lt, int l0, uint32_t* planes,
                                  int64_t pwords, uint64_t* masks, int32_t* stats, int num_sms, bool* done,
                                  cudaStream_t st) {
  *done = false;
  int cl = 0, clusters = 0;
  AliasGroups ag;
  size_t smem = 0;
  if (!alias_cluster_plan<DM, FAST>(lt, n, l0, lt.nlat, cl, ag, clusters, smem)) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl * clusters, 1, 1);
  cfg.blockDim = dim3(ACT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  prof_mark(PROF_ALIAS, true, st);
  cudaError_t e = cudaLaunchKernelEx(&cfg, alias_cluster_kernel<DM, FAST>, freqs, n, lt, ag, planes, pwords);
  if (e != cudaSuccess) {  // e.g. a cluster shape the context cannot place: the L2-atomic kernels
    (void)cudaGetLastError();
    prof_mark(PROF_ALIAS, false, st);
    return 0;
  }
  int64_t want = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms * 8;
  const int blocks = (int)(want < cap ? want : cap);
  alias_planes_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(n, l0, lt.nlat, planes, pwords, masks, stats);
  prof_mark(PROF_ALIAS, false, st);
  SFFT_CHECK_LAUNCHES(2);
  *done = true;
  return 0;
}

// ---------------------------------------------------------------------------
// Counter variant (default when the lattices' 32-bit counters, 4 sum M bytes,
// stay well inside L2): every (candidate, lattice) adds 1 to its residue's
// counter with a reduction that returns nothing (RED: the SM does not wait
// for the L2 round trip, where the bitmap variant needs the old word back to
// detect a second hit), and a candidate is alias-free on a lattice when its
// counter is exactly 1.  Same masks as the bitmaps for any multiplicity.
constexpr int64_t ALIAS_COUNTER_MAX_BYTES = 32ll << 20;

static bool alias_counters_enabled() {
  static const bool v = [] {
    const char* e = getenv("SFFT_B200_ALIAS_COUNTERS");
    return !(e && strcmp(e, "0") == 0);
  }();
  return v;
}

bool alias_counters_for(const int64_t* m, int L) {
  if (!alias_counters_enabled()) return false;
  int64_t tot = 0;
  for (int l = 0; l < L; ++l) tot += m[l];
  return 4 * tot <= ALIAS_COUNTER_MAX_BYTES;
}

template <int DM, bool FAST>
__global__ void __launch_bounds__(256)
alias_count_kernel(const int32_t* __restrict__ freqs, int64_t n, LatTable lt, int l0, uint32_t* __restrict__ cnt) {
  __shared__ int64_t co[SFFT_LMAX + 1];
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int l = 0; l < lt.nlat; ++l) { co[l] = acc; acc += lt.m[l]; }
    co[lt.nlat] = acc;
  }
  __syncthreads();
  const int d = lt.d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t k[DM];
    load_cand<DM>(k, freqs, n, i, d);
    for (int lb = l0; lb < lt.nlat; lb += AB) {
#pragma unroll
      for (int j = 0; j < AB; ++j) {
        const int l = lb + j;
        if (l < lt.nlat) atomicAdd(&cnt[co[l] + SFFT_RES(DM, FAST, k, lt, l)], 1u);  // RED, no return
      }
    }
  }
}

template <int DM, bool FAST>
__global__ void __launch_bounds__(256)
alias_cmask_kernel(const int32_t* __restrict__ freqs, int64_t n, LatTable lt, int l0,
                   const uint32_t* __restrict__ cnt, uint64_t* __restrict__ masks, int32_t* __restrict__ stats) {
  __shared__ int64_t co[SFFT_LMAX + 1];
  __shared__ int red[32];
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int l = 0; l < lt.nlat; ++l) { co[l] = acc; acc += lt.m[l]; }
    co[lt.nlat] = acc;
  }
  __syncthreads();
  const int d = lt.d;
  int first_max = 0, empty = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t k[DM];
    load_cand<DM>(k, freqs, n, i, d);
    uint64_t mask = l0 > 0 ? masks[i] : 0ull;
    for (int lb = l0; lb < lt.nlat; lb += AB) {
      uint32_t c[AB];
#pragma unroll
      for (int j = 0; j < AB; ++j) {  // the group's loads in flight together
        const int l = lb + j;
        c[j] = 0u;
        if (l < lt.nlat) c[j] = __ldg(&cnt[co[l] + SFFT_RES(DM, FAST, k, lt, l)]);
      }
#pragma unroll
      for (int j = 0; j < AB; ++j)
        if (c[j] == 1u) mask |= (1ull << (lb + j));
    }
    masks[i] = mask;
    if (mask) first_max = max(first_max, __ffsll((long long)mask));
    else empty += 1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    first_max = max(first_max, __shfl_down_sync(0xffffffffu, first_max, o));
    empty += __shfl_down_sync(0xffffffffu, empty, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { red[wid] = first_max; red[16 + wid] = empty; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int fm = 0, em = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { fm = max(fm, red[w]); em += red[16 + w]; }
    if (fm) atomicMax(&stats[0], fm);
    if (em) atomicAdd(&stats[1], em);
  }
}

int64_t alias_scratch_words(const LatTable& lt) {
  int64_t acc = 0;
  for (int l = 0; l < lt.nlat; ++l) acc += (lt.m[l] + 31) >> 5;
  return 2 * acc;
}

template <int DM, bool FAST>
static void launch_alias_t(const int32_t* freqs, int64_t n, const LatTable& lt, int l0, uint32_t* bits,
                           int64_t words, uint64_t* masks, int32_t* stats, int blocks,
                           cudaStream_t st) {
  prof_mark(PROF_ALIAS, true, st);
  alias_mark_kernel<DM, FAST><<<blocks, 256, 0, st>>>(freqs, n, lt, l0, bits, bits + words / 2, words);
  alias_mask_kernel<DM, FAST><<<blocks, 256, 0, st>>>(freqs, n, lt, l0, bits + words / 2, masks, stats);
  prof_mark(PROF_ALIAS, false, st);
}

// Lattices [l0, lt.nlat) of the table (l0 > 0: the masks of [0, l0) are in
// `masks` already); `words` = bitmap scratch of all lt.nlat lattices.
int launch_alias(const int32_t* freqs, int64_t n, const LatTable& lt, int l0, uint32_t* bits,
                 int64_t words, int64_t capacity, uint64_t* masks, int32_t* stats, bool fast, int num_sms,
                 cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(stats, 0, 2 * sizeof(int32_t), st);
  if (e != cudaSuccess) return (int)e;
  if (n == 0) return 0;
  const int d = lt.d;
  // cluster path: the scratch holds the alias-free bit-planes of the launch's
  // lattices (nlat - l0 planes of ceil(n / 32) words; always within the
  // bitmap scratch, since every M_l >= 2 |J| - 1)
  const int64_t pwords = (n + 31) >> 5;
  if ((int64_t)(lt.nlat - l0) * pwords <= words) {
    bool done = false;
    int rc = 0;
#define SFFT_ALIASC_CASE(DMV)                                                                              \
    if (d <= DMV) {                                                                                        \
      rc = fast ? launch_alias_cluster_t<DMV, true>(freqs, n, lt, l0, bits, pwords, masks, stats, num_sms, &done, st) \
                : launch_alias_cluster_t<DMV, false>(freqs, n, lt, l0, bits, pwords, masks, stats, num_sms, &done, st); \
    } else
    SFFT_ALIASC_CASE(4)
    SFFT_ALIASC_CASE(8)
    SFFT_ALIASC_CASE(16)
    SFFT_ALIASC_CASE(32)
    SFFT_ALIASC_CASE(64)
    { return -22; }
#undef SFFT_ALIASC_CASE
    if (rc) return rc;
    if (done) return 0;
  }
  int64_t want = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms * 8;
  int blocks = (int)(want < cap ? want : cap);
  if (alias_counters_for(lt.m, lt.nlat)) {
    int64_t c0 = 0, c1 = 0;
    for (int l = 0; l < lt.nlat; ++l) {
      if (l < l0) c0 += lt.m[l];
      c1 += lt.m[l];
    }
    if (c1 <= capacity) {
      // counters of lattices [l0, nlat) zeroed; [0, l0) belong to an earlier chunk
      e = cudaMemsetAsync(bits + c0, 0, (size_t)(c1 - c0) * sizeof(uint32_t), st);
      if (e != cudaSuccess) return (int)e;
#define SFFT_ALIASN_CASE(DMV)                                                                                    \
      if (d <= DMV) {                                                                                            \
        prof_mark(PROF_ALIAS, true, st);                                                                         \
        if (fast) {                                                                                              \
          alias_count_kernel<DMV, true><<<blocks, 256, 0, st>>>(freqs, n, lt, l0, bits);                         \
          alias_cmask_kernel<DMV, true><<<blocks, 256, 0, st>>>(freqs, n, lt, l0, bits, masks, stats);           \
        } else {                                                                                                 \
          alias_count_kernel<DMV, false><<<blocks, 256, 0, st>>>(freqs, n, lt, l0, bits);                        \
          alias_cmask_kernel<DMV, false><<<blocks, 256, 0, st>>>(freqs, n, lt, l0, bits, masks, stats);          \
        }                                                                                                        \
        prof_mark(PROF_ALIAS, false, st);                                                                        \
        SFFT_CHECK_LAUNCHES(2);                                                                                  \
        return 0;                                                                                                \
      }
      SFFT_ALIASN_CASE(4)
      SFFT_ALIASN_CASE(8)
      SFFT_ALIASN_CASE(16)
      SFFT_ALIASN_CASE(32)
      SFFT_ALIASN_CASE(64)
#undef SFFT_ALIASN_CASE
      return -22;
    }
  }
  e = cudaMemsetAsync(bits, 0, (size_t)words * sizeof(uint32_t), st);
  if (e != cudaSuccess) return (int)e;
#define SFFT_ALIAS_CASE(DMV)                                                                 \
  if (d <= DMV) {                                                                            \
    if (fast) launch_alias_t<DMV, true>(freqs, n, lt, l0, bits, words, masks, stats, blocks, st); \
    else launch_alias_t<DMV, false>(freqs, n, lt, l0, bits, words, masks, stats, blocks, st);     \
    SFFT_CHECK_LAUNCHES(2);                                                                  \
    return 0;                                                                                \
  }
  SFFT_ALIAS_CASE(4)
  SFFT_ALIAS_CASE(8)
  SFFT_ALIAS_CASE(16)
  SFFT_ALIAS_CASE(32)
  SFFT_ALIAS_CASE(64)
#undef SFFT_ALIAS_CASE
  return -22;  // EINVAL: dimension too large
}

}  // namespace sfft
