// K4: alias-free bin gather + lattice averaging + delta threshold, cap
// selection, stable compaction and the candidate product (K5).
//
// Reference: transform.py:99-127 (invert_multiple: spectrum_hat = fft / M,
// sums[mask] += spectrum_hat[res] in lattice order, coeffs = sums / counts),
// detect.py:197-212 (_select: |c| >= delta, cap by (|c| desc, freq lex asc)),
// detect.py:257-260 + 367-371 (candidate product), detect.py:412 and
// lattice.py:97-109 (union + lexsort/unique of the kept sets).
//
// numpy evaluates complex / int as a multiplication by the reciprocal
// (Smith's algorithm with a zero imaginary part), so the kernels do the same:
// spec * (1.0 / M) and sums * (1.0 / count).
//
// Candidate sets stay lexicographically sorted on the device without any
// sort: the product of a sorted prefix set with a sorted component set in
// row-major order is sorted, and every later set is an order-preserving
// subset of it (compaction by flags), so the reference's lexsort + unique
// reduces to a stable prefix-sum compaction.
#include "common.cuh"
#include "plan.cuh"
#include "gather.cuh"

namespace sfft {

template <int DM, bool FAST, int RB>
__global__ void __launch_bounds__(256)
gather_kernel(const int32_t* __restrict__ freqs, int64_t n, LatTable lt,
              const uint64_t* __restrict__ masks, const double2* __restrict__ buf, int64_t ustride,
              int rb, int it0, double delta, double2* __restrict__ coef, uint8_t* __restrict__ keep,
              int32_t* __restrict__ counts) {
  __shared__ int red[RB][8];
  const int d = lt.d;
  const int L = lt.nlat;
  const uint64_t lmask = (L >= 64) ? ~0ull : ((1ull << L) - 1ull);
  int kept[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) kept[i] = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t mask = masks[k] & lmask;
    double2 sums[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) sums[i] = make_double2(0.0, 0.0);
    int cnt = 0;
    if (mask) {
      int32_t kv[DM];
      load_cand<DM>(kv, freqs, n, k, d);
      uint64_t mm = mask;
      while (mm) {
        const int l = __ffsll((long long)mm) - 1;
        mm &= mm - 1;
        const int64_t r = SFFT_RES(DM, FAST, kv, lt, l);
        const double invm = lt.inv_m[l];  // == 1.0 / M (host-computed, correctly rounded)
        ++cnt;
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          if (i < rb) {
            // spectrum_hat = X / M rounded, then accumulated (no FMA contraction),
            // exactly the numpy sequence of transform.py:121-123
            const double2 v = __ldg(&buf[(int64_t)(i * L + l) * ustride + r]);
            sums[i].x = __dadd_rn(sums[i].x, __dmul_rn(v.x, invm));
            sums[i].y = __dadd_rn(sums[i].y, __dmul_rn(v.y, invm));
          }
        }
      }
    }
    const double invc = cnt ? 1.0 / (double)cnt : 0.0;
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      if (i < rb) {
        double2 c = make_double2(__dmul_rn(sums[i].x, invc), __dmul_rn(sums[i].y, invc));
        uint8_t kf = 0;
        if (cnt) {
          const double mag = hypot(c.x, c.y);
          kf = (mag >= delta) ? 1 : 0;
        } else {
          c = make_double2(0.0, 0.0);
        }
        coef[(int64_t)(it0 + i) * n + k] = c;
        keep[(int64_t)(it0 + i) * n + k] = kf;
        kept[i] += kf;
      }
    }
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
    int t = 0;
    for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
    if (t) atomicAdd(&counts[it0 + threadIdx.x], t);
  }
}

template <int DM, bool FAST>
static int launch_gather_t(const int32_t* freqs, int64_t n, const LatTable& lt,
                           const uint64_t* masks, const double2* buf, int64_t ustride, int rb,
                           int it0, double delta, double2* coef, uint8_t* keep, int32_t* counts,
                           int blocks, cudaStream_t st) {
  prof_mark(PROF_GATHER, true, st);
  if (rb <= 1)
    gather_kernel<DM, FAST, 1><<<blocks, 256, 0, st>>>(freqs, n, lt, masks, buf, ustride, rb, it0,
                                                       delta, coef, keep, counts);
  else if (rb <= 4)
    gather_kernel<DM, FAST, 4><<<blocks, 256, 0, st>>>(freqs, n, lt, masks, buf, ustride, rb, it0,
                                                       delta, coef, keep, counts);
  else if (rb <= 8)
    gather_kernel<DM, FAST, 8><<<blocks, 256, 0, st>>>(freqs, n, lt, masks, buf, ustride, rb, it0,
                                                       delta, coef, keep, counts);
  else
    return -22;
  prof_mark(PROF_GATHER, false, st);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_gather(const int32_t* freqs, int64_t n, const LatTable& lt, const uint64_t* masks,
                  const double2* buf, int64_t ustride, int rb, int it0, double delta, double2* coef,
                  uint8_t* keep, int32_t* counts, bool fast, int num_sms, cudaStream_t st) {
  if (n == 0) return 0;
  int64_t want = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms * 8;
  const int blocks = (int)(want < cap ? want : cap);
  const int d = lt.d;
#define SFFT_G_CASE(DMV)                                                                         \
  if (d <= DMV)                                                                                  \
    return fast ? launch_gather_t<DMV, true>(freqs, n, lt, masks, buf, ustride, rb, it0, delta, \
                                             coef, keep, counts, blocks, st)                    \
                : launch_gather_t<DMV, false>(freqs, n, lt, masks, buf, ustride, rb, it0, delta, \
                                              coef, keep, counts, blocks, st);
  SFFT_G_CASE(4)
  SFFT_G_CASE(8)
  SFFT_G_CASE(16)
  SFFT_G_CASE(32)
  SFFT_G_CASE(64)
#undef SFFT_G_CASE
  return -22;
}

// ---------------------------------------------------------------------------
// Sharded step (several GPUs): each rank gathers the alias-free bins of its
// own (iteration, lattice) units into dense per-unit rows
//     out[j][k] = bit l(j) of mask_k ? X_j[k.z_l mod M_l] * (1/M_l) : 0,
// the rows of all ranks are all-gathered (NCCL), and every rank combines them
// in lattice order with the same rounding sequence as gather_kernel, so the
// result is bit-identical for any number of GPUs.

template <int DM, bool FAST>
__global__ void __launch_bounds__(256)
gather_units_kernel(const int32_t* __restrict__ freqs, int64_t n, LatTable lt,
                    const uint64_t* __restrict__ masks, const double2* __restrict__ buf,
                    int64_t ustride, UnitTable ut, double2* __restrict__ out) {
  const int d = lt.d;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t mask = masks[k];
    int32_t kv[DM];
    load_cand<DM>(kv, freqs, n, k, d);
    for (int j = 0; j < ut.nunits; ++j) {
      const int l = ut.lat[j];
      double2 t = make_double2(0.0, 0.0);
      if ((mask >> l) & 1ull) {
        const int64_t r = SFFT_RES(DM, FAST, kv, lt, l);
        const double invm = lt.inv_m[l];  // == 1.0 / M (host-computed, correctly rounded)
        const double2 v = __ldg(&buf[(int64_t)j * ustride + r]);
        t = make_double2(__dmul_rn(v.x, invm), __dmul_rn(v.y, invm));
      }
      out[(int64_t)j * n + k] = t;
    }
  }
}

template <int RB>
__global__ void __launch_bounds__(256)
combine_units_kernel(int64_t n, int L, const uint64_t* __restrict__ masks,
                     const double2* __restrict__ vals, RowMap rm, int rb, int it0, double delta,
                     double2* __restrict__ coef, uint8_t* __restrict__ keep,
                     int32_t* __restrict__ counts) {
  __shared__ int red[RB][8];
  const uint64_t lmask = (L >= 64) ? ~0ull : ((1ull << L) - 1ull);
  int kept[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) kept[i] = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    uint64_t mm = masks[k] & lmask;
    double2 sums[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) sums[i] = make_double2(0.0, 0.0);
    int cnt = 0;
    while (mm) {
      const int l = __ffsll((long long)mm) - 1;
      mm &= mm - 1;
      ++cnt;
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        if (i < rb) {
          const double2 t = vals[(int64_t)rm.row[(it0 + i) * L + l] * n + k];
          sums[i].x = __dadd_rn(sums[i].x, t.x);
          sums[i].y = __dadd_rn(sums[i].y, t.y);
        }
      }
    }
    const double invc = cnt ? 1.0 / (double)cnt : 0.0;
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      if (i < rb) {
        double2 c = make_double2(__dmul_rn(sums[i].x, invc), __dmul_rn(sums[i].y, invc));
        uint8_t kf = 0;
        if (cnt) kf = (hypot(c.x, c.y) >= delta) ? 1 : 0;
        else c = make_double2(0.0, 0.0);
        coef[(int64_t)(it0 + i) * n + k] = c;
        keep[(int64_t)(it0 + i) * n + k] = kf;
        kept[i] += kf;
      }
    }
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
    int t = 0;
    for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
    if (t) atomicAdd(&counts[it0 + threadIdx.x], t);
  }
}

int launch_gather_units(const int32_t* freqs, int64_t n, const LatTable& lt, const uint64_t* masks,
                        const double2* buf, int64_t ustride, const UnitTable& ut, double2* out,
                        bool fast, int num_sms, cudaStream_t st) {
  if (n == 0 || ut.nunits == 0) return 0;
  int64_t want = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms * 8;
  const int blocks = (int)(want < cap ? want : cap);
  const int d = lt.d;
#define SFFT_GU_CASE(DMV)                                                                      \
  if (d <= DMV) {                                                                              \
    if (fast) gather_units_kernel<DMV, true><<<blocks, 256, 0, st>>>(freqs, n, lt, masks, buf, \
                                                                     ustride, ut, out);        \
    else gather_units_kernel<DMV, false><<<blocks, 256, 0, st>>>(freqs, n, lt, masks, buf,     \
                                                                 ustride, ut, out);            \
    SFFT_CHECK_LAUNCH();                                                                       \
    return 0;                                                                                  \
  }
  SFFT_GU_CASE(4)
  SFFT_GU_CASE(8)
  SFFT_GU_CASE(16)
  SFFT_GU_CASE(32)
  SFFT_GU_CASE(64)
#undef SFFT_GU_CASE
  return -22;
}

int launch_combine_units(int64_t n, int L, const uint64_t* masks, const double2* vals,
                         const RowMap& rm, int rb, int it0, double delta, double2* coef,
                         uint8_t* keep, int32_t* counts, int num_sms, cudaStream_t st) {
  if (n == 0) return 0;
  int64_t want = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms * 8;
  const int blocks = (int)(want < cap ? want : cap);
  if (rb <= 1)
    combine_units_kernel<1><<<blocks, 256, 0, st>>>(n, L, masks, vals, rm, rb, it0, delta, coef, keep, counts);
  else if (rb <= 4)
    combine_units_kernel<4><<<blocks, 256, 0, st>>>(n, L, masks, vals, rm, rb, it0, delta, coef, keep, counts);
  else if (rb <= 8)
    combine_units_kernel<8><<<blocks, 256, 0, st>>>(n, L, masks, vals, rm, rb, it0, delta, coef, keep, counts);
  else
    return -22;
  SFFT_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// flag -> ascending index list (stable compaction).  Flags of `nrows` rows of
// length n are OR-ed (union of the kept sets of several iterations).

constexpr int SCAN_T = 256;
constexpr int SCAN_PER = 1;  // one element per thread: n = 65000 gives 254 CTAs (8 per thread gave 32 CTAs, ~12 us each pass)
constexpr int SCAN_TILE = SCAN_T * SCAN_PER;

__device__ __forceinline__ int flag_at(const uint8_t* __restrict__ flags, int64_t n, int nrows, int64_t i) {
  int f = 0;
  for (int r = 0; r < nrows; ++r) f |= flags[(int64_t)r * n + i];
  return f != 0;
}

__global__ void scan_count_kernel(const uint8_t* __restrict__ flags, int64_t n, int nrows,
                                  int32_t* __restrict__ bcount) {
  __shared__ int red[32];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int c = 0;
  for (int q = 0; q < SCAN_PER; ++q) {
    const int64_t i = base + q * SCAN_T + threadIdx.x;
    if (i < n) c += flag_at(flags, n, nrows, i);
  }
  const int tot = block_sum(c, red);
  if (threadIdx.x == 0) bcount[blockIdx.x] = tot;
}

// single-block exclusive scan of nb block counts; total -> *total
__global__ void scan_blocks_kernel(int32_t* __restrict__ bcount, int64_t nb, int32_t* __restrict__ total) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t b0 = 0; b0 < nb; b0 += blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    int v = (i < nb) ? bcount[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = (lane < (int)(blockDim.x >> 5)) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;  // inclusive
    }
    __syncthreads();
    const int wbase = wid ? warp_tot[wid - 1] : 0;
    const int excl = carry + wbase + x - v;
    if (i < nb) bcount[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void scan_write_kernel(const uint8_t* __restrict__ flags, int64_t n, int nrows,
                                  const int32_t* __restrict__ boff, int32_t* __restrict__ idx_out) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = boff[blockIdx.x];
  __syncthreads();
  for (int q = 0; q < SCAN_PER; ++q) {
    const int64_t i = base + q * SCAN_T + threadIdx.x;
    const int v = (i < n) ? flag_at(flags, n, nrows, i) : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = (lane < (SCAN_T >> 5)) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;
    }
    __syncthreads();
    const int wbase = wid ? warp_tot[wid - 1] : 0;
    const int pos = carry + wbase + x - v;
    if (v) idx_out[pos] = (int32_t)i;
    __syncthreads();
    if (threadIdx.x == SCAN_T - 1) carry = pos + v;
    __syncthreads();
  }
}

int64_t scan_scratch_len(int64_t n) { return (n + SCAN_TILE - 1) / SCAN_TILE + 1; }

int launch_flag_indices(const uint8_t* flags, int64_t n, int nrows, int32_t* idx_out,
                        int32_t* total, int32_t* scratch, cudaStream_t st) {
  if (n == 0) {
    cudaError_t e = cudaMemsetAsync(total, 0, sizeof(int32_t), st);
    return (int)e;
  }
  const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  scan_count_kernel<<<(unsigned)nb, SCAN_T, 0, st>>>(flags, n, nrows, scratch);
  SFFT_CHECK_LAUNCH();
  scan_blocks_kernel<<<1, 1024, 0, st>>>(scratch, nb, total);
  SFFT_CHECK_LAUNCH();
  scan_write_kernel<<<(unsigned)nb, SCAN_T, 0, st>>>(flags, n, nrows, scratch, idx_out);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// rows: out[c * out_stride + j] = in[c * n_in + idx[j]] for j < *count (bounded by cap_rows)
__global__ void gather_rows_kernel(const int32_t* __restrict__ in, int64_t n_in, int ncomp,
                                   const int32_t* __restrict__ idx, const int32_t* __restrict__ count,
                                   int64_t cap_rows, int32_t* __restrict__ out, int64_t out_stride,
                                   const double2* __restrict__ cin, double2* __restrict__ cout) {
  const int64_t cnt = *count < cap_rows ? *count : cap_rows;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cnt;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t src = idx[j];
    for (int c = 0; c < ncomp; ++c) out[(int64_t)c * out_stride + j] = in[(int64_t)c * n_in + src];
    if (cout) cout[j] = cin[src];
  }
}

// covered[i] = (masks[i] != 0): the coverage flags of a scheme (the union of
// the reconstructing sets, MultipleRank1Lattice coverage) as bytes, 8 per thread
__global__ void masks_covered_kernel(const uint64_t* __restrict__ masks, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 8; i0 < n;
       i0 += (int64_t)gridDim.x * blockDim.x * 8) {
    if (i0 + 8 <= n) {
      uint64_t packed = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) packed |= (uint64_t)(masks[i0 + k] != 0ull ? 1 : 0) << (8 * k);
      *(uint64_t*)(out + i0) = packed;  // out is 8-byte aligned (caller's buffer start, i0 % 8 == 0)
    } else {
      for (int64_t i = i0; i < n; ++i) out[i] = masks[i] != 0ull ? 1 : 0;
    }
  }
}

int launch_masks_covered(const uint64_t* masks, int64_t n, uint8_t* out, int num_sms, cudaStream_t st) {
  if (n <= 0) return 0;
  int64_t want = (n + 8 * 256 - 1) / (8 * 256);
  const int64_t cap = (int64_t)num_sms * 8;
  masks_covered_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(masks, n, out);
  SFFT_CHECK_LAUNCH();
  return 0;
}

int launch_gather_rows(const int32_t* in, int64_t n_in, int ncomp, const int32_t* idx,
                       const int32_t* count, int64_t cap_rows, int32_t* out, int64_t out_stride,
                       const double2* cin, double2* cout, int num_sms, cudaStream_t st) {
  if (cap_rows <= 0) return 0;
  int64_t want = (cap_rows + 255) / 256;
  int64_t cap = (int64_t)num_sms * 8;
  gather_rows_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(
      in, n_in, ncomp, idx, count, cap_rows, out, out_stride, cin, cout);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// cap selection (detect.py:205-211): keep the `cap` largest |c| among the
// flagged entries, ties broken by ascending index (= ascending lexicographic
// frequency, since candidate sets are sorted).  Exact radix select on the
// IEEE bit pattern of |c| (monotone for non-negative doubles), 8 digits of 8
// bits, followed by an index-ordered rank among the entries equal to the
// threshold key.
struct SelState {
  unsigned long long prefix;
  unsigned long long pmask;
  int need;
  int pad;
};

__device__ __forceinline__ unsigned long long mag_key(double2 c) {
  return (unsigned long long)__double_as_longlong(hypot(c.x, c.y));
}

__global__ void sel_init_kernel(SelState* stt, int cap, int32_t* hist) {
  if (threadIdx.x == 0) { stt->prefix = 0; stt->pmask = 0; stt->need = cap; }
  hist[threadIdx.x] = 0;
}

__global__ void sel_hist_kernel(const double2* __restrict__ coef, const uint8_t* __restrict__ keep,
                                int64_t n, const SelState* __restrict__ stt, int shift,
                                int32_t* __restrict__ hist) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const unsigned long long pre = stt->prefix, pm = stt->pmask;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[i]) continue;
    const unsigned long long key = mag_key(coef[i]);
    if ((key & pm) != pre) continue;
    atomicAdd(&h[(key >> shift) & 255ull], 1);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// pick the digit holding the need-th largest key; clears hist for the next pass
__global__ void sel_pick_kernel(SelState* stt, int shift, int32_t* hist) {
  __shared__ int hs[256];
  hs[threadIdx.x] = hist[threadIdx.x];
  __syncthreads();
  hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    int need = stt->need;
    int above = 0;
    int dsel = 0;
    for (int dg = 255; dg >= 0; --dg) {
      if (above + hs[dg] >= need) { dsel = dg; break; }
      above += hs[dg];
    }
    stt->prefix |= ((unsigned long long)dsel) << shift;
    stt->pmask |= 255ull << shift;
    stt->need = need - above;
  }
}

// keep <- key > T ; tie flags for key == T
__global__ void sel_apply_kernel(const double2* __restrict__ coef, uint8_t* __restrict__ keep,
                                 int64_t n, const SelState* __restrict__ stt, uint8_t* __restrict__ tie) {
  const unsigned long long T = stt->prefix;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint8_t t = 0;
    if (keep[i]) {
      const unsigned long long key = mag_key(coef[i]);
      if (key == T) t = 1;
      keep[i] = (key > T) ? 1 : 0;
    }
    tie[i] = t;
  }
}

__global__ void sel_ties_kernel(uint8_t* __restrict__ keep, const int32_t* __restrict__ tie_idx,
                                const int32_t* __restrict__ ntie, const SelState* __restrict__ stt) {
  const int need = stt->need;
  const int nt = *ntie;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < need && j < nt; j += gridDim.x * blockDim.x)
    keep[tie_idx[j]] = 1;
}

int64_t select_scratch_bytes(int64_t n) {
  // state (64 B) + hist (1 KB) + tie flags (n) + tie idx (4n) + scan scratch + total
  return 64 + 1024 + ((n + 15) / 16) * 16 + 4 * n + 4 * scan_scratch_len(n) + 16;
}

int launch_select_cap(const double2* coef, uint8_t* keep, int64_t n, int cap, uint8_t* scratch,
                      int num_sms, cudaStream_t st) {
  if (n == 0) return 0;
  SelState* stt = (SelState*)scratch;
  int32_t* hist = (int32_t*)(scratch + 64);
  uint8_t* tie = scratch + 64 + 1024;
  int32_t* tie_idx = (int32_t*)(scratch + 64 + 1024 + ((n + 15) / 16) * 16);
  int32_t* sscr = tie_idx + n;
  int32_t* total = sscr + scan_scratch_len(n);
  int64_t want = (n + 255) / 256;
  int64_t capb = (int64_t)num_sms * 4;
  const unsigned blocks = (unsigned)(want < capb ? want : capb);
  sel_init_kernel<<<1, 256, 0, st>>>(stt, cap, hist);
  SFFT_CHECK_LAUNCH();
  for (int dgt = 7; dgt >= 0; --dgt) {
    const int shift = dgt * 8;
    sel_hist_kernel<<<blocks, 256, 0, st>>>(coef, keep, n, stt, shift, hist);
    sel_pick_kernel<<<1, 256, 0, st>>>(stt, shift, hist);
  }
  SFFT_CHECK_LAUNCHES(16);
  sel_apply_kernel<<<blocks, 256, 0, st>>>(coef, keep, n, stt, tie);
  SFFT_CHECK_LAUNCH();
  int rc = launch_flag_indices(tie, n, 1, tie_idx, total, sscr, st);
  if (rc) return rc;
  sel_ties_kernel<<<blocks, 256, 0, st>>>(keep, tie_idx, total, stt);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// Batched cap selection: several iterations (rows of coef/keep) at once, the
// histogram and the digit pick of each radix pass fused (the last CTA of a
// row to finish its histogram picks the digit), ties resolved by one CTA per
// row with a block scan in index order.  11 launches per step instead of
// ~22 per capped iteration; identical selection to launch_select_cap.
struct SelRows {
  int nrows;
  int row[64];
};

constexpr int SEL_TIE_LIST = 2048;  // tie entries resolved by rank in shared memory

struct SelRowState {
  unsigned long long prefix, pmask;
  int need, done;  // done: CTAs finished with the current pass
  int count_eq;    // entries whose key equals the threshold (after the last pass)
  int nlist;       // tie entries appended by selr_apply
  int active;      // the row's survivor count exceeds the cap (device-side decision)
  int hist[256];
  int list[SEL_TIE_LIST];
};

// d_counts (optional): survivor counts per row of keep; rows not above the cap
// are left untouched by every later kernel, capped rows get count = cap
__global__ void selr_init_kernel(SelRowState* st, int cap, SelRows rows, int32_t* counts) {
  SelRowState& s = st[blockIdx.x];
  if (threadIdx.x == 0) {
    s.prefix = 0; s.pmask = 0; s.need = cap; s.done = 0; s.count_eq = 0; s.nlist = 0;
    s.active = 1;
    if (counts) {
      const int c = counts[rows.row[blockIdx.x]];
      s.active = c > cap;
      if (s.active) counts[rows.row[blockIdx.x]] = cap;
    }
  }
  s.hist[threadIdx.x] = 0;
}

__global__ void selr_pass_kernel(const double2* __restrict__ coef, const uint8_t* __restrict__ keep, int64_t n,
                                 SelRows rows, SelRowState* st, int shift) {
  __shared__ int h[256];
  __shared__ bool last;
  const int y = blockIdx.y;
  SelRowState& s = st[y];
  if (!s.active) return;
  const double2* c = coef + (int64_t)rows.row[y] * n;
  const uint8_t* k = keep + (int64_t)rows.row[y] * n;
  h[threadIdx.x] = 0;
  __syncthreads();
  const unsigned long long pre = s.prefix, pm = s.pmask;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!k[i]) continue;
    const unsigned long long key = mag_key(c[i]);
    if ((key & pm) != pre) continue;
    atomicAdd(&h[(key >> shift) & 255ull], 1);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&s.hist[threadIdx.x], h[threadIdx.x]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&s.done, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  // last CTA of this row: pick the digit holding the need-th largest key
  __threadfence();
  h[threadIdx.x] = atomicExch(&s.hist[threadIdx.x], 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    int need = s.need, above = 0, dsel = 0;
    for (int dg = 255; dg >= 0; --dg) {
      if (above + h[dg] >= need) { dsel = dg; break; }
      above += h[dg];
    }
    s.prefix |= ((unsigned long long)dsel) << shift;
    s.pmask |= 255ull << shift;
    s.need = need - above;
    s.count_eq = h[dsel];
    s.done = 0;
  }
}

// keep <- key > T; entries with key == T: all kept when they are exactly the
// `need` still missing, otherwise marked 2 and listed for selr_ties
__global__ void selr_apply_kernel(const double2* __restrict__ coef, uint8_t* __restrict__ keep, int64_t n,
                                  SelRows rows, SelRowState* st) {
  const int y = blockIdx.y;
  SelRowState& s = st[y];
  if (!s.active) return;
  const unsigned long long T = s.prefix;
  const bool all_ties = s.count_eq == s.need;
  const double2* c = coef + (int64_t)rows.row[y] * n;
  uint8_t* k = keep + (int64_t)rows.row[y] * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!k[i]) continue;
    const unsigned long long key = mag_key(c[i]);
    if (key == T && !all_ties) {
      const int pos = atomicAdd(&s.nlist, 1);
      if (pos < SEL_TIE_LIST) s.list[pos] = (int)i;
      k[i] = 2;
    } else {
      k[i] = key >= T ? 1 : 0;
    }
  }
}

// one CTA per row: the first `need` tie entries in index order are kept
// (rank within the appended list; overflowed lists: the chunked kernels below)
__global__ void __launch_bounds__(1024) selr_ties_kernel(uint8_t* __restrict__ keep, int64_t n, SelRows rows,
                                                         const SelRowState* __restrict__ st) {
  __shared__ int lst[SEL_TIE_LIST];
  const SelRowState& s = st[blockIdx.x];
  if (!s.active || s.count_eq == s.need) return;  // nothing capped, or every tie kept in selr_apply
  uint8_t* k = keep + (int64_t)rows.row[blockIdx.x] * n;
  const int need = s.need;
  const int nl = s.nlist;
  if (nl <= SEL_TIE_LIST) {
    for (int j = threadIdx.x; j < nl; j += blockDim.x) lst[j] = s.list[j];
    __syncthreads();
    for (int j = threadIdx.x; j < nl; j += blockDim.x) {
      const int v = lst[j];
      int rank = 0;
      for (int q = 0; q < nl; ++q) rank += lst[q] < v;
      k[v] = rank < need ? 1 : 0;
    }
    return;
  }
  // more ties than the list holds: selr_tiecount / selr_tiescan / selr_tiemark
}

// Overflowed tie lists (more than SEL_TIE_LIST entries equal to the threshold,
// e.g. the +-k mirror ties of the B-spline spectrum at a binding cap): ranks
// in index order by a chunked count / scan / mark over all CTAs; the row's
// list storage holds the per-chunk counts (at most SEL_TIE_LIST chunks).
__host__ __device__ inline int64_t tie_chunk(int64_t n) {
  const int64_t per = (n + SEL_TIE_LIST - 1) / SEL_TIE_LIST;
  return ((per + 2047) / 2048) * 2048;
}

__device__ __forceinline__ bool tie_overflow(const SelRowState& s) {
  return s.active && s.count_eq != s.need && s.nlist > SEL_TIE_LIST;
}

__global__ void __launch_bounds__(256) selr_tiecount_kernel(const uint8_t* __restrict__ keep, int64_t n,
                                                            SelRows rows, SelRowState* st) {
  __shared__ int red[8];
  SelRowState& s = st[blockIdx.y];
  if (!tie_overflow(s)) return;
  const int64_t ch = tie_chunk(n);
  const int64_t i0 = (int64_t)blockIdx.x * ch, i1 = min(n, i0 + ch);
  const uint8_t* k = keep + (int64_t)rows.row[blockIdx.y] * n;
  int c = 0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) c += k[i] == 2;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    s.list[blockIdx.x] = t;
  }
}

__global__ void selr_tiescan_kernel(int64_t n, SelRowState* st) {
  SelRowState& s = st[blockIdx.x];
  if (!tie_overflow(s) || threadIdx.x != 0) return;
  const int nch = (int)((n + tie_chunk(n) - 1) / tie_chunk(n));
  int acc = 0;
  for (int c = 0; c < nch; ++c) {
    const int v = s.list[c];
    s.list[c] = acc;
    acc += v;
  }
}

__global__ void __launch_bounds__(256) selr_tiemark_kernel(uint8_t* __restrict__ keep, int64_t n, SelRows rows,
                                                           const SelRowState* __restrict__ st) {
  __shared__ int wsum[8];
  const SelRowState& s = st[blockIdx.y];
  if (!tie_overflow(s)) return;
  const int64_t ch = tie_chunk(n);
  const int64_t i0 = (int64_t)blockIdx.x * ch, i1 = min(n, i0 + ch);
  uint8_t* k = keep + (int64_t)rows.row[blockIdx.y] * n;
  const int need = s.need;
  int base = s.list[blockIdx.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t b = i0; b < i1; b += blockDim.x) {
    const int64_t i = b + threadIdx.x;
    const bool t = i < i1 && k[i] == 2;
    const unsigned bal = __ballot_sync(0xffffffffu, t);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      before += j < w ? wsum[j] : 0;
      total += wsum[j];
    }
    if (t) k[i] = (base + before + __popc(bal & ((1u << lane) - 1u))) < need ? 1 : 0;
    base += total;
    __syncthreads();
  }
}

int64_t select_rows_scratch_bytes(int nrows) { return (int64_t)nrows * sizeof(SelRowState); }

int launch_select_cap_rows(const double2* coef, uint8_t* keep, int64_t n, const int32_t* h_rows, int nrows,
                           int cap, int32_t* counts, uint8_t* scratch, int num_sms, cudaStream_t st) {
  if (n == 0 || nrows == 0) return 0;
  if (nrows > 64) return -7;
  SelRows rows;
  rows.nrows = nrows;
  for (int i = 0; i < nrows; ++i) rows.row[i] = h_rows[i];
  SelRowState* s = (SelRowState*)scratch;
  int64_t want = (n + 255) / 256;
  int64_t capb = ((int64_t)num_sms * 4 + nrows - 1) / nrows;
  const unsigned blocks = (unsigned)(want < capb ? want : capb);
  selr_init_kernel<<<nrows, 256, 0, st>>>(s, cap, rows, counts);
  for (int dgt = 7; dgt >= 0; --dgt)
    selr_pass_kernel<<<dim3(blocks, nrows), 256, 0, st>>>(coef, keep, n, rows, s, dgt * 8);
  selr_apply_kernel<<<dim3(blocks, nrows), 256, 0, st>>>(coef, keep, n, rows, s);
  selr_ties_kernel<<<nrows, 1024, 0, st>>>(keep, n, rows, s);
  const unsigned nch = (unsigned)((n + tie_chunk(n) - 1) / tie_chunk(n));
  selr_tiecount_kernel<<<dim3(nch, nrows), 256, 0, st>>>(keep, n, rows, s);
  selr_tiescan_kernel<<<nrows, 32, 0, st>>>(n, s);
  selr_tiemark_kernel<<<dim3(nch, nrows), 256, 0, st>>>(keep, n, rows, s);
  SFFT_CHECK_LAUNCHES(14);
  return 0;
}

// ---------------------------------------------------------------------------
// candidate product (detect.py:257-260): row q = a * nc + b  ->  (prefix_a, comp_b)
__global__ void product_kernel(const int32_t* __restrict__ pref, int64_t np, int t,
                               const int32_t* __restrict__ comp, int64_t nc, int32_t* __restrict__ out) {
  const int64_t total = np * nc;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = q / nc, b = q - a * nc;
    for (int c = 0; c < t; ++c) out[(int64_t)c * total + q] = pref[(int64_t)c * np + a];
    out[(int64_t)t * total + q] = comp[b];
  }
}

int launch_product(const int32_t* pref, int64_t np, int t, const int32_t* comp, int64_t nc,
                   int32_t* out, int num_sms, cudaStream_t st) {
  const int64_t total = np * nc;
  if (total == 0) return 0;
  int64_t want = (total + 255) / 256;
  int64_t cap = (int64_t)num_sms * 16;
  product_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(pref, np, t, comp, nc, out);
  SFFT_CHECK_LAUNCH();
  return 0;
}

// residues k.z_l mod M_l of every candidate on every lattice: out[l * n + i]
template <int DM, bool FAST>
__global__ void residues_kernel(const int32_t* __restrict__ freqs, int64_t n, LatTable lt,
                                int64_t* __restrict__ out) {
  const int d = lt.d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t k[DM];
    load_cand<DM>(k, freqs, n, i, d);
    for (int l = 0; l < lt.nlat; ++l)
      out[(int64_t)l * n + i] = SFFT_RES(DM, FAST, k, lt, l);
  }
}

int launch_residues(const int32_t* freqs, int64_t n, const LatTable& lt, int64_t* out, bool fast,
                    int num_sms, cudaStream_t st) {
  if (n == 0) return 0;
  int64_t want = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms * 8;
  const unsigned blocks = (unsigned)(want < cap ? want : cap);
  const int d = lt.d;
#define SFFT_R_CASE(DMV)                                                                     \
  if (d <= DMV) {                                                                            \
    if (fast) residues_kernel<DMV, true><<<blocks, 256, 0, st>>>(freqs, n, lt, out);         \
    else residues_kernel<DMV, false><<<blocks, 256, 0, st>>>(freqs, n, lt, out);             \
    SFFT_CHECK_LAUNCH();                                                                     \
    return 0;                                                                                \
  }
  SFFT_R_CASE(4)
  SFFT_R_CASE(8)
  SFFT_R_CASE(16)
  SFFT_R_CASE(32)
  SFFT_R_CASE(64)
#undef SFFT_R_CASE
  return -22;
}

// Host rows (n x d int64, row-major, as numpy hands them over) -> the
// component-major int32 device layout, with per-component min / max
// (minmax[c] = min, minmax[d + c] = max) and an out-of-range flag
// (minmax[2d] = 1 if some |k| > 2^31 - 1, lattice.py:36-38).
__global__ void pack_rows_init_kernel(int d, int32_t* __restrict__ minmax) {
  const int c = threadIdx.x;
  if (c < d) { minmax[c] = INT32_MAX; minmax[d + c] = INT32_MIN; }
  if (c == 0) minmax[2 * d] = 0;
}

__global__ void pack_rows_kernel(const int64_t* __restrict__ rows, int64_t n, int d,
                                 int32_t* __restrict__ out, int32_t* __restrict__ minmax) {
  __shared__ int smin[SFFT_DMAX], smax[SFFT_DMAX];
  for (int c = threadIdx.x; c < d; c += blockDim.x) { smin[c] = INT32_MAX; smax[c] = INT32_MIN; }
  __syncthreads();
  const int64_t total = n * d;
  int bad = 0;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = rows[f];
    const int64_t i = f / d;
    const int c = (int)(f - i * d);
    if (v > 2147483647LL || v < -2147483647LL) bad = 1;
    const int32_t w = (int32_t)v;
    out[(int64_t)c * n + i] = w;
    atomicMin(&smin[c], w);
    atomicMax(&smax[c], w);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    atomicMin(&minmax[c], smin[c]);
    atomicMax(&minmax[d + c], smax[c]);
  }
  if (bad) atomicOr(&minmax[2 * d], 1);
}

int launch_pack_rows(const int64_t* rows, int64_t n, int d, int32_t* out, int32_t* minmax,
                     int num_sms, cudaStream_t st) {
  if (d < 1 || d > SFFT_DMAX) return -22;
  pack_rows_init_kernel<<<1, 64, 0, st>>>(d, minmax);
  SFFT_CHECK_LAUNCH();
  if (n == 0) return 0;
  int64_t want = (n * d + 255) / 256;
  int64_t cap = (int64_t)num_sms * 8;
  pack_rows_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(rows, n, d, out, minmax);
  SFFT_CHECK_LAUNCH();
  return 0;
}

__global__ void cscale_kernel(double2* __restrict__ x, int64_t n, double scale, int conj) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = x[i];
    if (conj) v.y = -v.y;
    x[i] = make_double2(v.x * scale, v.y * scale);
  }
}

int launch_cscale(double2* x, int64_t n, double scale, int conj, int num_sms, cudaStream_t st) {
  if (n == 0) return 0;
  int64_t want = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms * 8;
  cscale_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(x, n, scale, conj);
  SFFT_CHECK_LAUNCH();
  return 0;
}

}  // namespace sfft
