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
#include "common.cuh"
#include "plan.cuh"

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
#pragma unroll
    for (int c = 0; c < DM; ++c) k[c] = (c < d) ? __ldg(&freqs[(int64_t)c * n + i]) : 0;
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
#pragma unroll
    for (int c = 0; c < DM; ++c) k[c] = (c < d) ? __ldg(&freqs[(int64_t)c * n + i]) : 0;
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
                 int64_t words, uint64_t* masks, int32_t* stats, bool fast, int num_sms,
                 cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(bits, 0, (size_t)words * sizeof(uint32_t), st);
  if (e != cudaSuccess) return (int)e;
  e = cudaMemsetAsync(stats, 0, 2 * sizeof(int32_t), st);
  if (e != cudaSuccess) return (int)e;
  if (n == 0) return 0;
  int64_t want = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms * 8;
  int blocks = (int)(want < cap ? want : cap);
  const int d = lt.d;
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
