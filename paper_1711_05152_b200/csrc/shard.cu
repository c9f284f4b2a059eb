// Sliced exchange of a sharded MR1L step.
//
// The (iteration, lattice) units of a step are dealt round-robin over the G
// ranks; candidates are cut into G contiguous slices of whole 256-candidate
// tiles.  Rank g owns slice g of the result.  Every rank
//   1. packs, for each of its units (lattice l) and each slice q, the
//      alias-free bins X_u[k.z_l mod M_l] * (1/M_l) of the slice's candidates
//      whose mask bit l is set, in candidate order (sfft_pack_units),
//   2. exchanges the packs with one all-to-all (NCCL over NVLink; the packs
//      hold only alias-free entries, ~0.61 |J| per unit, and each rank
//      receives only its slice: |J| * sum_l 0.61 * 16 B / G per iteration),
//   3. combines its slice in lattice order with exactly the rounding sequence
//      of the single-GPU gather (transform.py:118-124: spectrum * (1/M),
//      summed l = 1..L, times 1/count) and thresholds it (sfft_combine_slice),
//   4. all-gathers the keep flags (and the coefficients when the step needs
//      them: the last step, or a binding cap) and reassembles them
//      (sfft_unshard_rows).
// The position of candidate k's entry in a pack is its rank among the
// slice's candidates with bit l set: a per-tile / per-lattice popcount table
// scanned along the tiles (sfft_mask_tiles) plus a ballot prefix in the tile.
// Results are bit-identical for any G (and to run_step on one GPU).
#include "common.cuh"
#include "plan.cuh"

namespace sfft {

constexpr int TT = 256;  // candidates per tile (one CTA)

// popcount of mask bit l over tile t: tc[t * L + l]
__global__ void __launch_bounds__(TT) tile_counts_kernel(const uint64_t* __restrict__ masks, int64_t n, int L,
                                                         int64_t ntiles, int32_t* __restrict__ tc) {
  __shared__ int ws[TT / 32][SFFT_LMAX];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t k = t * TT + threadIdx.x;
    const uint64_t m = k < n ? masks[k] : 0ull;
    for (int l = 0; l < L; ++l) {
      const unsigned bal = __ballot_sync(0xffffffffu, (m >> l) & 1ull);
      if (lane == 0) ws[w][l] = __popc(bal);
    }
    __syncthreads();
    for (int l = threadIdx.x; l < L; l += TT) {
      int s = 0;
#pragma unroll
      for (int q = 0; q < TT / 32; ++q) s += ws[q][l];
      tc[t * L + l] = s;
    }
    __syncthreads();
  }
}

// exclusive scan along the tiles, one CTA per lattice:
// toff[t * L + l] = sum_{t' < t} tc[t' * L + l], t = 0 .. ntiles;
// slice totals sc[q * L + l] for slices of ts tiles
__global__ void __launch_bounds__(TT) tile_scan_kernel(const int32_t* __restrict__ tc, int64_t ntiles, int L,
                                                       int32_t* __restrict__ toff, int64_t ts, int W,
                                                       int32_t* __restrict__ sc) {
  __shared__ int wsum[TT / 32];
  const int l = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int running = 0;
  for (int64_t b = 0; b < ntiles; b += TT) {
    const int64_t t = b + threadIdx.x;
    const int v = t < ntiles ? tc[t * L + l] : 0;
    int x = v;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int q = 0; q < TT / 32; ++q) {
      before += q < w ? wsum[q] : 0;
      total += wsum[q];
    }
    if (t < ntiles) toff[t * L + l] = running + before + x - v;
    running += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) toff[ntiles * L + l] = running;
  __syncthreads();
  __threadfence_block();
  for (int q = threadIdx.x; q < W; q += TT) {
    const int64_t a = min(ntiles, (int64_t)q * ts), e = min(ntiles, (int64_t)(q + 1) * ts);
    sc[q * L + l] = toff[e * L + l] - toff[a * L + l];
  }
}

// per-warp ballots of every lattice bit of a tile and their warp prefixes
struct TileRanks {
  unsigned bal[TT / 32][SFFT_LMAX];
  int pre[TT / 32][SFFT_LMAX];
};

__device__ __forceinline__ void tile_ranks(TileRanks& tr, uint64_t m, int L) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int l = 0; l < L; ++l) {
    const unsigned bal = __ballot_sync(0xffffffffu, (m >> l) & 1ull);
    if (lane == 0) tr.bal[w][l] = bal;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < L; l += TT) {
    int s = 0;
#pragma unroll
    for (int q = 0; q < TT / 32; ++q) {
      tr.pre[q][l] = s;
      s += __popc(tr.bal[q][l]);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ int rank_in_tile(const TileRanks& tr, int l) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  return tr.pre[w][l] + __popc(tr.bal[w][l] & ((1u << lane) - 1u));
}

// pack the own units' alias-free bins, slice-major: unit slot j's entries of
// slice q start at soff[q * nown + j]
template <int DM, bool FAST>
__global__ void __launch_bounds__(TT)
pack_units_kernel(const int32_t* __restrict__ freqs, int64_t n, LatTable lt, const uint64_t* __restrict__ masks,
                  const double2* __restrict__ buf, int64_t ustride, UnitTable ut,
                  const int32_t* __restrict__ toff, int64_t ntiles, int64_t ts,
                  const int64_t* __restrict__ soff, double2* __restrict__ send) {
  __shared__ TileRanks tr;
  const int L = lt.nlat;
  const int d = lt.d;
  const uint64_t lmask = (L >= 64) ? ~0ull : ((1ull << L) - 1ull);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t k = t * TT + threadIdx.x;
    const uint64_t m = k < n ? (masks[k] & lmask) : 0ull;
    tile_ranks(tr, m, L);
    const int q = (int)(t / ts);
    const int64_t t0 = (int64_t)q * ts;
    if (m) {
      int32_t kv[DM];
      load_cand<DM>(kv, freqs, n, k, d);
      int lprev = -1;
      int64_t r = 0;
      for (int j = 0; j < ut.nunits; ++j) {
        const int l = ut.lat[j];
        if (!((m >> l) & 1ull)) continue;
        if (l != lprev) {
          r = SFFT_RES(DM, FAST, kv, lt, l);
          lprev = l;
        }
        const int64_t pos = soff[(int64_t)q * ut.nunits + j] + (toff[t * L + l] - toff[t0 * L + l]) +
                            rank_in_tile(tr, l);
        const double invm = lt.inv_m[l];
        const double2 v = __ldg(&buf[(int64_t)j * ustride + r]);
        send[pos] = make_double2(__dmul_rn(v.x, invm), __dmul_rn(v.y, invm));
      }
    }
    __syncthreads();
  }
}

// combine slice q (lattice order, the single-GPU rounding), threshold;
// outputs [rb][S] for the slice's candidates (S = ts tiles * TT), survivor
// counts of the slice added into counts[i]
template <int RB>
__global__ void __launch_bounds__(TT)
combine_slice_kernel(int64_t n, int L, const uint64_t* __restrict__ masks, const int32_t* __restrict__ toff,
                     int64_t ntiles, int64_t ts, int q, const double2* __restrict__ recv,
                     const int64_t* __restrict__ roff, int rb, double delta, double2* __restrict__ coef_s,
                     uint8_t* __restrict__ keep_s, int32_t* __restrict__ counts) {
  __shared__ TileRanks tr;
  __shared__ int red[RB][TT / 32];
  const uint64_t lmask = (L >= 64) ? ~0ull : ((1ull << L) - 1ull);
  const int64_t t0 = (int64_t)q * ts, t1 = min(ntiles, t0 + ts);
  const int64_t S = ts * TT;
  int kept[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) kept[i] = 0;
  for (int64_t t = t0 + blockIdx.x; t < t1; t += gridDim.x) {
    const int64_t k = t * TT + threadIdx.x;
    const bool live = k < n;
    const uint64_t m = live ? (masks[k] & lmask) : 0ull;
    tile_ranks(tr, m, L);
    double2 sums[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) sums[i] = make_double2(0.0, 0.0);
    int cnt = 0;
    uint64_t mm = m;
    while (mm) {
      const int l = __ffsll((long long)mm) - 1;
      mm &= mm - 1;
      ++cnt;
      const int64_t rank = (toff[t * L + l] - toff[t0 * L + l]) + rank_in_tile(tr, l);
#pragma unroll
      for (int i = 0; i < RB; ++i)
        if (i < rb) {
          const double2 v = __ldg(&recv[roff[i * L + l] + rank]);
          sums[i].x = __dadd_rn(sums[i].x, v.x);
          sums[i].y = __dadd_rn(sums[i].y, v.y);
        }
    }
    if (live) {
      const double invc = cnt ? 1.0 / (double)cnt : 0.0;
      const int64_t sidx = k - t0 * TT;
#pragma unroll
      for (int i = 0; i < RB; ++i)
        if (i < rb) {
          double2 c = make_double2(__dmul_rn(sums[i].x, invc), __dmul_rn(sums[i].y, invc));
          uint8_t kf = 0;
          if (cnt) kf = hypot(c.x, c.y) >= delta ? 1 : 0;
          else c = make_double2(0.0, 0.0);
          coef_s[(int64_t)i * S + sidx] = c;
          keep_s[(int64_t)i * S + sidx] = kf;
          kept[i] += kf;
        }
    }
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    int v = kept[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[i][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < RB && threadIdx.x < rb) {
    int s = 0;
    for (int w = 0; w < TT / 32; ++w) s += red[threadIdx.x][w];
    if (s) atomicAdd(&counts[threadIdx.x], s);
  }
}

// [W][rb][S] slice-major rows (all-gathered) -> rows it0 .. it0 + rb - 1 of
// [r][n]; elem = 1 (keep flags) or 16 (coefficients) bytes
template <typename T>
__global__ void unshard_kernel(const T* __restrict__ in, int W, int rb, int64_t S, int64_t n, int it0,
                               T* __restrict__ out) {
  const int64_t total = (int64_t)rb * n;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / n, k = x - i * n;
    const int64_t q = k / S, s = k - q * S;
    out[(int64_t)(it0 + i) * n + k] = in[(q * rb + i) * S + s];
  }
}

// ---------------------------------------------------------------------------
// launchers

int launch_mask_tiles(const uint64_t* masks, int64_t n, int L, int32_t* tc, int32_t* toff, int64_t ts, int W,
                      int32_t* sc, int num_sms, cudaStream_t st) {
  if (L < 1 || L > SFFT_LMAX || W < 1 || ts < 1) return -22;
  const int64_t ntiles = (n + TT - 1) / TT;
  if (ntiles > 0) {
    const int64_t cap = (int64_t)num_sms * 8;
    tile_counts_kernel<<<(unsigned)(ntiles < cap ? ntiles : cap), TT, 0, st>>>(masks, n, L, ntiles, tc);
    SFFT_CHECK_LAUNCH();
  }
  tile_scan_kernel<<<L, TT, 0, st>>>(tc, ntiles, L, toff, ts, W, sc);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_pack_units(const int32_t* freqs, int64_t n, const LatTable& lt, const uint64_t* masks,
                      const double2* buf, int64_t ustride, const UnitTable& ut, const int32_t* toff, int64_t ts,
                      const int64_t* soff, double2* send, bool fast, int num_sms, cudaStream_t st) {
  const int64_t ntiles = (n + TT - 1) / TT;
  if (ntiles == 0 || ut.nunits == 0) return 0;
  const int64_t cap = (int64_t)num_sms * 8;
  const unsigned blocks = (unsigned)(ntiles < cap ? ntiles : cap);
  const int d = lt.d;
#define SFFT_PK_CASE(DMV)                                                                                  \
  if (d <= DMV) {                                                                                          \
    if (fast) pack_units_kernel<DMV, true><<<blocks, TT, 0, st>>>(freqs, n, lt, masks, buf, ustride, ut,  \
                                                                  toff, ntiles, ts, soff, send);           \
    else pack_units_kernel<DMV, false><<<blocks, TT, 0, st>>>(freqs, n, lt, masks, buf, ustride, ut, toff, \
                                                              ntiles, ts, soff, send);                     \
    SFFT_CHECK_LAUNCH();                                                                                   \
    return 0;                                                                                              \
  }
  SFFT_PK_CASE(4)
  SFFT_PK_CASE(8)
  SFFT_PK_CASE(16)
  SFFT_PK_CASE(32)
  SFFT_PK_CASE(64)
#undef SFFT_PK_CASE
  return -22;
}

int launch_combine_slice(int64_t n, int L, const uint64_t* masks, const int32_t* toff, int64_t ts, int q,
                         const double2* recv, const int64_t* roff, int rb, double delta, double2* coef_s,
                         uint8_t* keep_s, int32_t* counts, int num_sms, cudaStream_t st) {
  const int64_t ntiles = (n + TT - 1) / TT;
  const int64_t mine = min(ntiles, (int64_t)(q + 1) * ts) - min(ntiles, (int64_t)q * ts);
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)rb, st);
  if (e != cudaSuccess) return (int)e;
  if (mine <= 0) return 0;
  const int64_t cap = (int64_t)num_sms * 8;
  const unsigned blocks = (unsigned)(mine < cap ? mine : cap);
#define SFFT_CS(RBV) \
  combine_slice_kernel<RBV><<<blocks, TT, 0, st>>>(n, L, masks, toff, ntiles, ts, q, recv, roff, rb, delta, coef_s, \
                                                   keep_s, counts)
  if (rb <= 1) SFFT_CS(1);
  else if (rb <= 4) SFFT_CS(4);
  else if (rb <= 8) SFFT_CS(8);
  else return -22;
#undef SFFT_CS
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_unshard(const void* in, int elem, int W, int rb, int64_t S, int64_t n, int it0, void* out, int num_sms,
                   cudaStream_t st) {
  const int64_t total = (int64_t)rb * n;
  if (total == 0) return 0;
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = (int64_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  if (elem == 1)
    unshard_kernel<uint8_t><<<(unsigned)blocks, 256, 0, st>>>((const uint8_t*)in, W, rb, S, n, it0, (uint8_t*)out);
  else if (elem == 16)
    unshard_kernel<double2><<<(unsigned)blocks, 256, 0, st>>>((const double2*)in, W, rb, S, n, it0, (double2*)out);
  else
    return -22;
  SFFT_CHECK_LAUNCH();
  return 0;
}

}  // namespace sfft
