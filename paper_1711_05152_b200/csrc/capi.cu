// extern "C" boundary (include/sfft_b200.h): validates arguments, builds the
// by-value launch structs and dispatches to the kernels.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <unordered_map>

#include "../../include/sfft_b200.h"
#include "common.cuh"
#include "gather.cuh"
#include "lines.cuh"
#include "plan.cuh"
#include "sample.cuh"

namespace sfft {
int launch_cbc_scan(const int64_t* prefix_res, const int32_t* col, int64_t n, int64_t m, int64_t z0,
                    int Z, uint32_t* bits, int64_t words, int32_t* dup, int num_sms, cudaStream_t st);
int launch_prefix_flags(const int32_t* freqs, int64_t n, int t1, uint8_t* flags, int num_sms,
                        cudaStream_t st);
int launch_scatter_residues(const int32_t* freqs, int64_t n, const LatTable& lt, const double2* coef,
                            double2* acc, int num_sms, cudaStream_t st);
int launch_fp64_peak(double* out, int iters, int blocks, cudaStream_t st);
int launch_mask_tiles(const uint64_t* masks, int64_t n, int L, int32_t* tc, int32_t* toff, int64_t ts, int W,
                      int32_t* sc, int num_sms, cudaStream_t st);
int launch_pack_units(const int32_t* freqs, int64_t n, const LatTable& lt, const uint64_t* masks,
                      const double2* buf, int64_t ustride, const UnitTable& ut, const int32_t* toff, int64_t ts,
                      const int64_t* soff, double2* send, bool fast, int num_sms, cudaStream_t st);
int launch_combine_slice(int64_t n, int L, const uint64_t* masks, const int32_t* toff, int64_t ts, int q,
                         const double2* recv, const int64_t* roff, int rb, double delta, double2* coef_s,
                         uint8_t* keep_s, int32_t* counts, int num_sms, cudaStream_t st);
int launch_unshard(const void* in, int elem, int W, int rb, int64_t S, int64_t n, int it0, void* out, int num_sms,
                   cudaStream_t st);
int launch_fp64_mma_peak(double* out, int iters, int blocks, cudaStream_t st);
int launch_l2_random_peak(uint32_t* bits, uint32_t words, int blocks, int per_thread, int mode, cudaStream_t st);
int launch_eval_poly_points(const double* pts, int64_t n, int d, const int32_t* hf,
                            const double2* coef, int s, double2* out, cudaStream_t st);
int launch_eval_bspline_points(const double* pts, int64_t n, const BsplineSpec& bs, double2* out,
                               int num_sms, cudaStream_t st);
int launch_line_points(const double* anchors, int d, int r, int K, double* pts, int num_sms, cudaStream_t st);
int launch_add_noise(double2* x, const double2* e, int64_t n, double scale, int num_sms,
                     cudaStream_t st);
}

using namespace sfft;

// ---------------------------------------------------------------------------
// kernel-class event profiling
namespace {
constexpr int PROF_RING = 4096;
struct ProfState {
  std::mutex mu;
  bool on = false;
  cudaEvent_t ev[PROF_NCLASS][PROF_RING][2];
  bool made[PROF_NCLASS][PROF_RING];
  int n[PROF_NCLASS];
  int open[PROF_NCLASS];
};
ProfState& prof() {
  static ProfState* p = [] {
    auto* q = new ProfState;
    memset(q->made, 0, sizeof(q->made));
    memset(q->n, 0, sizeof(q->n));
    memset(q->open, 0, sizeof(q->open));
    return q;
  }();
  return *p;
}
}  // namespace

namespace sfft {
void prof_mark(int cls, bool begin, cudaStream_t st) {
  ProfState& p = prof();
  if (!p.on) return;
  std::lock_guard<std::mutex> g(p.mu);
  int i = p.n[cls];
  if (i >= PROF_RING) return;
  if (!p.made[cls][i]) {
    cudaEventCreate(&p.ev[cls][i][0]);
    cudaEventCreate(&p.ev[cls][i][1]);
    p.made[cls][i] = true;
  }
  cudaEventRecord(p.ev[cls][i][begin ? 0 : 1], st);
  if (!begin) p.n[cls] = i + 1;
}
}  // namespace sfft

namespace {

constexpr int E_INVAL = -22;
constexpr int E_2BIG = -7;

int num_sms_current() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

int fill_lat(LatTable& lt, const int64_t* h_m, const int32_t* h_z, int L, int t1) {
  if (L < 0 || L > SFFT_LMAX) return E_2BIG;
  if (t1 < 0 || t1 > SFFT_DMAX || (int64_t)L * t1 > SFFT_ZMAX) return E_2BIG;
  memset(&lt, 0, sizeof(LatTable));
  lt.nlat = L;
  lt.d = t1;
  int64_t off = 0;
  for (int l = 0; l < L; ++l) {
    const int64_t m = h_m[l];
    if (m < 1 || m > 2147483647LL) return E_INVAL;
    lt.m[l] = m;
    lt.inv_m[l] = 1.0 / (double)m;
    lt.off[l] = off;
    off += m;
    if (h_z)
      for (int c = 0; c < t1; ++c) {
        int64_t zc = h_z[l * t1 + c];
        if (zc < 0 || zc >= m) return E_INVAL;
        lt.z[l * t1 + c] = (int32_t)zc;
      }
  }
  return 0;
}

// Units of a launch: all rb x L (iteration, lattice) pairs in order
// (h_units == NULL), or the explicit list h_units[j] = it * L + l (it < rb),
// buffer slot j holding unit h_units[j] (the sharded engine's local units).
int fill_units(UnitTable& ut, const int64_t* h_m, int L, int rb, const int32_t* h_units = nullptr,
               int nunits = 0) {
  if (L < 1 || L > SFFT_LMAX || rb < 1) return E_2BIG;
  const int nu = h_units ? nunits : rb * L;
  if (nu < 1 || nu > SFFT_UMAX) return E_2BIG;
  memset(&ut, 0, sizeof(UnitTable));
  ut.nunits = nu;
  ut.nlat = L;
  int64_t off = 0;
  for (int l = 0; l < L; ++l) {
    ut.m[l] = h_m[l];
    ut.off[l] = off;
    off += h_m[l];
  }
  for (int j = 0; j < nu; ++j) {
    const int g = h_units ? h_units[j] : j;
    if (g < 0 || g >= rb * L) return E_INVAL;
    ut.lat[j] = g % L;
    ut.it[j] = g / L;
  }
  return 0;
}

bool residue_fast(int t1, int64_t kmax, const int64_t* h_m, int L) {
  int64_t mmax = 1;
  for (int l = 0; l < L; ++l) mmax = h_m[l] > mmax ? h_m[l] : mmax;
  const double bound = (double)t1 * (double)(kmax < 0 ? -kmax : kmax) * (double)mmax;
  return bound < 4503599627370496.0;  // every |k . z| < 2^52: exact in a double, mod_fast's domain
}

// Enable the int32 residue path when every |k . z| < d * kmax * M < 2^31.
void set_i32(LatTable& lt, int64_t kmax) {
  int64_t mmax = 1;
  for (int l = 0; l < lt.nlat; ++l) mmax = lt.m[l] > mmax ? lt.m[l] : mmax;
  const double bound = (double)lt.d * (double)(kmax < 0 ? -kmax : kmax) * (double)mmax;
  lt.i32 = bound < 2147483647.0 ? 1 : 0;
  for (int l = 0; l < lt.nlat; ++l) {
    lt.mu32[l] = (uint32_t)(0xFFFFFFFFull / (uint64_t)lt.m[l]);
    lt.off32[l] = lt.i32 ? (uint32_t)(lt.m[l] * (int64_t)lt.d * (kmax < 0 ? -kmax : kmax)) : 0u;
  }
}

bool fast_i32(LatTable& lt, int t1, int64_t kmax, const int64_t* h_m, int L) {
  set_i32(lt, kmax);
  return residue_fast(t1, kmax, h_m, L);
}

bool mulmod_fast(const int64_t* h_m, int L) {
  int64_t mmax = 1;
  for (int l = 0; l < L; ++l) mmax = h_m[l] > mmax ? h_m[l] : mmax;
  const double b = (double)(mmax + 64) * (double)(mmax + 64);
  return b < 4.0e15;
}

int fill_bspline(BsplineSpec& bs, int ngroups, const int32_t* h_order, const int32_t* h_start,
                 const int32_t* h_comps, const double* h_scale, int d) {
  if (ngroups < 0 || ngroups > 8 || d < 1 || d > SFFT_DMAX) return E_INVAL;
  memset(&bs, 0, sizeof(bs));
  bs.d = d;
  bs.ngroups = ngroups;
  if (h_start[0] != 0 || h_start[ngroups] > SFFT_DMAX) return E_2BIG;
  for (int g = 0; g <= ngroups; ++g) bs.start[g] = h_start[g];
  for (int g = 0; g < ngroups; ++g) {
    if (h_order[g] < 1 || h_order[g] > 7 || h_start[g + 1] < h_start[g]) return E_INVAL;
    bs.order[g] = h_order[g];
    bs.scale[g] = h_scale[g];
  }
  for (int q = 0; q < h_start[ngroups]; ++q) {
    if (h_comps[q] < 0 || h_comps[q] >= d) return E_INVAL;
    bs.comps[q] = h_comps[q];
  }
  // pieces of B_m (testbed.py:198-216 evaluates the same spline with scipy's
  // BSpline.basis_element): P_1 = [1]; piece i of B_k in t = u - i is
  // ((t + i) P_{k-1,i}(t) + (k - i - t) P_{k-1,i-1}(t)) / (k - 1)
  double prev[8][8] = {{1.0}};
  bs.pc[bs_poff(1)] = 1.0;
  for (int k = 2; k <= 7; ++k) {
    double cur[8][8] = {};
    for (int i = 0; i < k; ++i) {
      for (int e = 0; e < k - 1; ++e) {  // degree of P_{k-1} is k - 2
        const double a = i < k - 1 ? prev[i][e] : 0.0;      // P_{k-1,i}
        const double b = i >= 1 ? prev[i - 1][e] : 0.0;      // P_{k-1,i-1}
        cur[i][e] += (double)i * a + (double)(k - i) * b;    // constant parts
        cur[i][e + 1] += a - b;                              // t * a - t * b
      }
      for (int e = 0; e < k; ++e) cur[i][e] /= (double)(k - 1);
    }
    for (int i = 0; i < k; ++i)
      for (int e = 0; e < k; ++e) bs.pc[bs_poff(k) + i * k + e] = cur[i][e];
    memcpy(prev, cur, sizeof(prev));
  }
  return 0;
}

// J1 (multiple of 64) minimising the padded tile count J1 * 64 * ceil(J2 / 64);
// memoised per M (the same primes recur across steps and calls)
void choose_j1_search(int64_t m, int& j1, int& nt1, int& nt2);

void choose_j1_search(int64_t m, int tw2, int& j1, int& nt1, int& nt2);

// tiles are 64 (j1) x tw2 (j2), tw2 = 64 (classic kernel) or 128 (warp-specialised)
void choose_j1(int64_t m, int tw2, int& j1, int& nt1, int& nt2) {
  static std::mutex mu;
  static std::unordered_map<int64_t, int> memo;
  const int64_t key = m * 2 + (tw2 == 128 ? 1 : 0);
  {
    std::lock_guard<std::mutex> g(mu);
    auto itr = memo.find(key);
    if (itr != memo.end()) {
      j1 = itr->second;
      nt1 = j1 / 64;
      const int64_t J2 = (m + j1 - 1) / j1;
      nt2 = (int)((J2 + tw2 - 1) / tw2);
      return;
    }
  }
  choose_j1_search(m, tw2, j1, nt1, nt2);
  std::lock_guard<std::mutex> g(mu);
  if (memo.size() > 65536) memo.clear();
  memo[key] = j1;
}

void choose_j1_search(int64_t m, int tw2, int& j1, int& nt1, int& nt2) {
  int64_t best = -1;
  int bj = 64;
  const int64_t amax = (m + 63) / 64;
  const int64_t alim = amax < 4096 ? amax : 4096;
  const double root = sqrt((double)m);
  // Among the least-padded factorisations the tensor-core kernel (tw2 = 128)
  // takes the widest J1: its B operand is precomputed per lattice as
  // ceil(J2 / 128) column tiles x all terms (poly_bpanel_kernel), so fewer
  // column tiles mean proportionally smaller panels (config 1: 5 -> 1 tiles,
  // ~25 -> ~5 MB per lattice, L2-resident for the contraction) for the same
  // padded node count.  The classic kernel keeps J1 near sqrt(M).
  static const bool wide = [] {
    const char* e = getenv("SFFT_B200_J1_WIDE");
    return !(e && strcmp(e, "0") == 0);
  }();
  const bool prefer_wide = wide && tw2 == 128;
  for (int64_t a = 1; a <= alim; ++a) {
    const int64_t J1 = 64 * a;
    const int64_t J2 = (m + J1 - 1) / J1;
    const int64_t padded = J1 * tw2 * ((J2 + tw2 - 1) / tw2);
    if (best < 0 || padded < best ||
        (padded == best && (prefer_wide ? J1 > bj : fabs((double)J1 - root) < fabs((double)bj - root)))) {
      best = padded;
      bj = (int)J1;
    }
  }
  j1 = bj;
  nt1 = bj / 64;
  const int64_t J2 = (m + bj - 1) / bj;
  nt2 = (int)((J2 + tw2 - 1) / tw2);
}

// polynomial sampling kernel: SFFT_B200_SAMPLE_KERNEL=classic|ws|tc
// (default tc: warp-specialised, FP64 tensor-core contraction)
int sample_kind() {
  static int kind = [] {
    const char* e = getenv("SFFT_B200_SAMPLE_KERNEL");
    if (e && strcmp(e, "classic") == 0) return 0;
    if (e && strcmp(e, "ws") == 0) return 1;
    return 2;
  }();
  return kind;
}

// Tiles, K split and table split of the GEMM-factored polynomial sampling.
// The K split (term slices reduced in order by a second kernel) is chosen to
// maximise the fraction of the last wave that is busy; `need` = partial-sum
// scratch in complex elements (0 without a split).  partial_cap < 0: unlimited.
int build_poly_plan(PolyPlan* pp, const int64_t* h_m, int L, const UnitTable& ut, int rb_hint, int s,
                    int num_sms, int64_t partial_cap, int64_t* need) {
  if (L < 1 || L > SFFT_LMAX || ut.nunits < 1 || ut.nunits > SFFT_UMAX || s < 0) return E_2BIG;
  memset(pp, 0, sizeof(PolyPlan));
  pp->nunits = ut.nunits;
  pp->s = s;
  int64_t mmax = 1;
  for (int l = 0; l < L; ++l) mmax = h_m[l] > mmax ? h_m[l] : mmax;
  int bl = 1;
  while (((int64_t)1 << (2 * bl)) < mmax) ++bl;
  pp->bl = bl;
  pp->kind = sample_kind();
  if (pp->kind >= 1 && sample_poly_ws_smem(bl, mmax) > 227 * 1024 - 256) pp->kind = 0;  // + static mbarriers
  const size_t smem = pp->kind >= 1 ? sample_poly_ws_smem(bl, mmax) : sample_poly_smem(bl, mmax);
  if (smem > 227 * 1024) return E_2BIG;
  // resident CTAs per SM: classic 2 by registers (256 threads x 128 regs),
  // warp-specialised 1 (384 threads x 168 regs); fewer if shared-memory-bound
  const int reg_cap = pp->kind >= 1 ? 1 : 2;
  int per_sm = (int)((228 * 1024) / (smem + 1024));
  if (per_sm > reg_cap) per_sm = reg_cap;
  if (per_sm < 1) per_sm = 1;
  const int tw2 = pp->kind >= 1 ? 128 : 64;
  int64_t tiles_l[SFFT_LMAX];
  int64_t tiles_total = 0;
  for (int l = 0; l < L; ++l) {
    int j1, nt1, nt2;
    choose_j1(h_m[l], tw2, j1, nt1, nt2);
    pp->J1[l] = j1;
    pp->nt1[l] = nt1;
    pp->nt2[l] = nt2;
    tiles_l[l] = (int64_t)nt1 * nt2;
    pp->mu[l] = ~0ull / (uint64_t)h_m[l];
  }
  // The K split is chosen for the full chunk of rb x L units even when this
  // launch holds a subset (sharded step): the term slicing, and so every
  // rounding, is then independent of the number of GPUs.
  int rb_nominal = 1;
  for (int u = 0; u < ut.nunits; ++u) rb_nominal = ut.it[u] + 1 > rb_nominal ? ut.it[u] + 1 : rb_nominal;
  if (rb_hint > rb_nominal) rb_nominal = rb_hint;
  for (int l = 0; l < L; ++l) tiles_total += (int64_t)rb_nominal * tiles_l[l];
  const int64_t slots = (int64_t)per_sm * num_sms;
  int best_ks = 1, best_kper = ((s + 15) / 16) * 16;
  double best_eff = -1.0;
  for (int ks = 1; ks <= 8; ++ks) {
    int kper = (((s + ks - 1) / ks + 15) / 16) * 16;
    if (kper < 16) kper = 16;
    const int kse = (s + kper - 1) / kper > 0 ? (s + kper - 1) / kper : 1;
    if (ks > 1 && (kper < 64 || kse != ks)) continue;
    if (kse > 1 && partial_cap >= 0 && (int64_t)kse * pp->nunits * mmax > partial_cap) continue;
    const int64_t units = tiles_total * kse;
    const int64_t waves = (units + slots - 1) / slots;
    double eff = (double)units / (double)(waves * slots);
    if (kse > 1) eff *= 0.97;  // partial-sum write/read + reduce kernel
    if (eff > best_eff + 1e-9) { best_eff = eff; best_ks = kse; best_kper = kper; }
  }
  static const int force_ks = [] {  // measurement override (tools): SFFT_B200_KSPLIT=<1..8>
    const char* e = getenv("SFFT_B200_KSPLIT");
    return e ? atoi(e) : 0;
  }();
  if (force_ks >= 1 && force_ks <= 8) {
    int kper = (((s + force_ks - 1) / force_ks + 15) / 16) * 16;
    if (kper < 16) kper = 16;
    const int kse = (s + kper - 1) / kper > 0 ? (s + kper - 1) / kper : 1;
    if (kse == 1 || partial_cap < 0 || (int64_t)kse * pp->nunits * mmax <= partial_cap) {
      best_kper = kper;
      best_ks = kse;
    }
  }
  pp->ks = best_ks;
  pp->kper = best_kper;
  int64_t acc = 0;
  for (int u = 0; u < ut.nunits; ++u) {
    pp->unit_lat[u] = ut.lat[u];
    pp->unit_it[u] = ut.it[u];
    pp->tile_start[u] = (int)acc;
    acc += tiles_l[ut.lat[u]] * best_ks;
  }
  pp->tile_start[ut.nunits] = (int)acc;
  if (acc > 0x7fffffffLL) return E_2BIG;
  const int64_t partials = best_ks > 1 ? (int64_t)best_ks * pp->nunits * mmax : 0;
  *need = partials;
  if (pp->kind == 2) {
    pp->nchunk_total = (s + 15) / 16;
    int64_t blocks = 0;
    for (int l = 0; l < L; ++l) {
      pp->panel_off[l] = (int)blocks;
      blocks += (int64_t)pp->nt2[l] * pp->nchunk_total;
    }
    if (blocks > 0x7fffffffLL / 2048) return E_2BIG;
    pp->npanels = (int)blocks;
    pp->partial_base = blocks * 2048;  // panels first (32 KB each), partial sums after
    *need = pp->partial_base + partials;
    if (best_ks > 1) {  // then the publish flags of the in-kernel reduction
      pp->flag_base = *need;
      *need += SFFT_WS_MAX_FLAGS * 4 / 16;
    }
  }
  return 0;
}

}  // namespace

extern "C" {

int sfft_abi_version(void) { return SFFT_B200_ABI_VERSION; }

long long sfft_launch_count(void) { return g_launches.load(); }

int sfft_profile_enable(int on) {
  ProfState& p = prof();
  std::lock_guard<std::mutex> g(p.mu);
  p.on = on != 0;
  memset(p.n, 0, sizeof(p.n));
  return 0;
}

int sfft_profile_collect(int cls, double* total_ms, int* count) {
  if (cls < 0 || cls >= PROF_NCLASS) return E_INVAL;
  ProfState& p = prof();
  std::lock_guard<std::mutex> g(p.mu);
  double tot = 0.0;
  for (int i = 0; i < p.n[cls]; ++i) {
    cudaError_t e = cudaEventSynchronize(p.ev[cls][i][1]);
    if (e != cudaSuccess) return (int)e;
    float ms = 0.f;
    e = cudaEventElapsedTime(&ms, p.ev[cls][i][0], p.ev[cls][i][1]);
    if (e != cudaSuccess) return (int)e;
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (count) *count = p.n[cls];
  p.n[cls] = 0;
  return 0;
}

const char* sfft_error_string(int code) {
  if (code == 0) return "ok";
  if (code == E_INVAL) return "invalid argument";
  if (code == E_2BIG) return "argument exceeds a device-table limit";
  if (code > 0) return cudaGetErrorString((cudaError_t)code);
  return "unknown error";
}

int sfft_device_info(int* num_sms, int* cc_major, int* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  if (num_sms) *num_sms = num_sms_current();
  if (cc_major) cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
  if (cc_minor) cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  return 0;
}

int sfft_copy_async(void* dst, const void* src, int64_t nbytes, void* stream) {
  if (nbytes < 0 || (nbytes > 0 && (!dst || !src))) return E_INVAL;
  if (nbytes == 0) return 0;
  return (int)cudaMemcpyAsync(dst, src, (size_t)nbytes, cudaMemcpyDefault, S(stream));
}

int64_t sfft_alias_scratch_words(const int64_t* h_m, int L) {
  int64_t acc = 0, tot = 0;
  for (int l = 0; l < L; ++l) {
    acc += (h_m[l] + 31) >> 5;
    tot += h_m[l];
  }
  // two bitmaps of the lattices, or their 32-bit counters (alias.cu counter variant)
  return alias_counters_for(h_m, L) && tot > 2 * acc ? tot : 2 * acc;
}

static int64_t alias_bitmap_words(const int64_t* h_m, int L) {
  int64_t acc = 0;
  for (int l = 0; l < L; ++l) acc += (h_m[l] + 31) >> 5;
  return 2 * acc;
}

int sfft_alias_masks_range(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax, const int64_t* h_m,
                           const int32_t* h_z, int l0, int l1, uint32_t* d_scratch, int64_t scratch_words,
                           uint64_t* d_masks, int32_t* d_stats, void* stream) {
  if (n < 0 || t1 < 1 || l0 < 0 || l1 <= l0) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, h_m, h_z, l1, t1);
  if (rc) return rc;
  const int64_t need = alias_bitmap_words(h_m, l1);  // the bitmaps always fit; counters when the scratch allows
  if (scratch_words < need) return E_INVAL;
  return launch_alias(d_freqs, n, lt, l0, d_scratch, need, scratch_words, d_masks, d_stats,
                      fast_i32(lt, t1, kmax, h_m, l1), num_sms_current(), S(stream));
}

int sfft_alias_masks(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax, const int64_t* h_m,
                     const int32_t* h_z, int L, uint32_t* d_scratch, int64_t scratch_words,
                     uint64_t* d_masks, int32_t* d_stats, void* stream) {
  if (L < 1) return E_INVAL;
  return sfft_alias_masks_range(d_freqs, n, t1, kmax, h_m, h_z, 0, L, d_scratch, scratch_words, d_masks,
                                d_stats, stream);
}

int sfft_lattice_tables(const int64_t* h_m, int L, double* d_tw, double* d_chirp, void* stream) {
  LatTable lt;
  int rc = fill_lat(lt, h_m, nullptr, L, 0);
  if (rc) return rc;
  if (L == 0) return 0;
  return launch_lattice_tables(lt, (double2*)d_tw, (double2*)d_chirp, S(stream));
}

static bool fft_pow2_only() {
  static const bool v = [] {
    const char* e = getenv("SFFT_B200_FFT_POW2");
    return e && strcmp(e, "1") == 0;
  }();
  return v;
}

int64_t sfft_fft_size(int64_t m_max) {
  if (m_max < 1) return -1;
  return fft_choose_size(m_max, fft_pow2_only());
}

int64_t sfft_fft_table_len(int64_t P) {
  const FftGeom g = fft_geom(P);
  return g.valid ? g.table_len : -1;
}

int sfft_fft_tables(int64_t P, double* d_ftab, void* stream) {
  const FftGeom g = fft_geom(P);
  if (!g.valid) return E_INVAL;
  return launch_fft_tables(g, (double2*)d_ftab, S(stream));
}

int sfft_bluestein_bhat(const int64_t* h_m, int L, int64_t P, const double* d_ftab,
                        const double* d_chirp, double* d_bhat, void* stream) {
  const FftGeom g = fft_geom(P);
  if (!g.valid) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, h_m, nullptr, L, 0);
  if (rc) return rc;
  for (int l = 0; l < L; ++l)
    if (2 * h_m[l] - 1 > P) return E_INVAL;
  return launch_bhat(lt, (const double2*)d_chirp, (double2*)d_bhat, g, (const double2*)d_ftab,
                     S(stream));
}

int sfft_bluestein(const int64_t* h_m, int L, int rb, int64_t P, const double* d_ftab,
                   const double* d_bhat, const double* d_chirp, double* d_buf,
                   const int32_t* h_units, int nunits, void* stream) {
  const FftGeom g = fft_geom(P);
  if (!g.valid) return E_INVAL;
  UnitTable ut;
  int rc = fill_units(ut, h_m, L, rb, h_units, nunits);
  if (rc) return rc;
  for (int l = 0; l < L; ++l)
    if (2 * h_m[l] - 1 > P) return E_INVAL;
  return launch_bluestein((double2*)d_buf, ut, g, (const double2*)d_ftab, (const double2*)d_bhat,
                          (const double2*)d_chirp, S(stream));
}

static int sample_poly_impl(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int t1,
                            const int64_t* h_m, const int32_t* h_z, int L, const double* h_anchor, int rb,
                            double* d_cprime, int32_t* d_rres, int32_t* d_rj, const double* d_tw,
                            const double* d_chirp, double* d_buf, int64_t P, int apply_chirp,
                            double* d_partial, int64_t partial_len, const int32_t* h_units, int nunits,
                            void* stream, bool do_prepare, bool do_run, bool panels_ready = false) {
  if (s < 0 || d < 1 || t1 < 1 || t1 > d || d > SFFT_DMAX || rb < 1) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, h_m, h_z, L, t1);
  if (rc) return rc;
  UnitTable ut;
  rc = fill_units(ut, h_m, L, rb, h_units, nunits);
  if (rc) return rc;
  const int tail = d - t1;
  if ((int64_t)rb * tail > SFFT_ANCHOR_MAX) return E_2BIG;
  AnchorTable at;
  at.rb = rb;
  at.tail = tail;
  for (int i = 0; i < rb * tail; ++i) at.a[i] = h_anchor[i];
  PolyPlan* pp = new PolyPlan;
  int64_t need = 0;
  rc = build_poly_plan(pp, h_m, L, ut, rb, s, num_sms_current(), partial_len, &need);
  if (rc) { delete pp; return rc; }
  if (need > partial_len) { delete pp; return E_2BIG; }  // scratch smaller than sfft_sample_poly_scratch
  int64_t mmax = 1;
  for (int l = 0; l < L; ++l) mmax = h_m[l] > mmax ? h_m[l] : mmax;
  cudaStream_t st = S(stream);
  if (do_prepare)
    rc = launch_poly_prepare(d_hfreqs, (const double2*)d_hcoef, s, d, lt, *pp, at,
                             (double2*)d_cprime, d_rres, d_rj, st);
  if (!rc && do_run)
    rc = launch_sample_poly(*pp, lt, ut, (const double2*)d_cprime, d_rres, d_rj,
                            (const double2*)d_tw, (const double2*)d_chirp, (double2*)d_buf, P,
                            apply_chirp != 0, (double2*)d_partial, mmax, num_sms_current(), st, panels_ready);
  delete pp;
  return rc;
}

int sfft_sample_poly(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int t1,
                     const int64_t* h_m, const int32_t* h_z, int L, const double* h_anchor, int rb,
                     double* d_cprime, int32_t* d_rres, int32_t* d_rj, const double* d_tw,
                     const double* d_chirp, double* d_buf, int64_t P, int apply_chirp,
                     double* d_partial, int64_t partial_len, const int32_t* h_units, int nunits,
                     void* stream) {
  return sample_poly_impl(d_hfreqs, d_hcoef, s, d, t1, h_m, h_z, L, h_anchor, rb, d_cprime, d_rres, d_rj, d_tw,
                          d_chirp, d_buf, P, apply_chirp, d_partial, partial_len, h_units, nunits, stream, true,
                          true);
}

int sfft_sample_poly_prepare(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int t1,
                             const int64_t* h_m, const int32_t* h_z, int L, const double* h_anchor, int rb,
                             double* d_cprime, int32_t* d_rres, int32_t* d_rj, const double* d_tw,
                             double* d_scratch, int64_t scratch_len, int* h_panels_built, void* stream) {
  if (h_panels_built) *h_panels_built = 0;
  if (s < 0 || d < 1 || t1 < 1 || t1 > d || d > SFFT_DMAX || rb < 1) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, h_m, h_z, L, t1);
  if (rc) return rc;
  UnitTable ut;
  rc = fill_units(ut, h_m, L, rb, nullptr, 0);
  if (rc) return rc;
  const int tail = d - t1;
  if ((int64_t)rb * tail > SFFT_ANCHOR_MAX) return E_2BIG;
  AnchorTable at;
  at.rb = rb;
  at.tail = tail;
  for (int i = 0; i < rb * tail; ++i) at.a[i] = h_anchor[i];
  PolyPlan* pp = new PolyPlan;
  int64_t need = 0;
  rc = build_poly_plan(pp, h_m, L, ut, rb, s, num_sms_current(), -1, &need);  // J1, panel layout
  if (!rc)
    rc = launch_poly_prepare(d_hfreqs, (const double2*)d_hcoef, s, d, lt, *pp, at, (double2*)d_cprime, d_rres,
                             d_rj, S(stream));
  // B panels of all L lattices (the K-split-independent region at the start of
  // the scratch) when a scratch and the lattice twiddles are given
  if (!rc && d_scratch && d_tw && pp->kind == 2 && (int64_t)pp->npanels * 2048 <= scratch_len) {
    rc = launch_bpanels(*pp, lt, d_rj, (const double2*)d_tw, d_scratch, S(stream));
    if (!rc && h_panels_built) *h_panels_built = 1;
  }
  delete pp;
  return rc;
}

int sfft_sample_poly_run(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int t1,
                         const int64_t* h_m, const int32_t* h_z, int L, const double* h_anchor, int rb,
                         double* d_cprime, int32_t* d_rres, int32_t* d_rj, const double* d_tw,
                         const double* d_chirp, double* d_buf, int64_t P, int apply_chirp,
                         double* d_partial, int64_t partial_len, const int32_t* h_units, int nunits,
                         int panels_ready, void* stream) {
  return sample_poly_impl(d_hfreqs, d_hcoef, s, d, t1, h_m, h_z, L, h_anchor, rb, d_cprime, d_rres, d_rj, d_tw,
                          d_chirp, d_buf, P, apply_chirp, d_partial, partial_len, h_units, nunits, stream, false,
                          true, panels_ready != 0);
}

int64_t sfft_sample_poly_scratch(const int64_t* h_m, int L, int rb, int s, const int32_t* h_units,
                                 int nunits) {
  UnitTable ut;
  if (fill_units(ut, h_m, L, rb, h_units, nunits)) return -1;
  PolyPlan* pp = new PolyPlan;
  int64_t need = 0;
  int rc = build_poly_plan(pp, h_m, L, ut, rb, s, num_sms_current(), -1, &need);
  delete pp;
  return rc ? -1 : need;
}

int sfft_sample_bspline(int ngroups, const int32_t* h_order, const int32_t* h_start,
                        const int32_t* h_comps, const double* h_scale, int d, int t1,
                        const int64_t* h_m, const int32_t* h_z, int L, const double* h_anchor,
                        int rb, const double* d_chirp, double* d_buf, int64_t P, int apply_chirp,
                        const int32_t* h_units, int nunits, void* stream) {
  if (ngroups < 0 || ngroups > 8 || d < 1 || d > SFFT_DMAX || t1 < 1 || t1 > d) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, h_m, h_z, L, t1);
  if (rc) return rc;
  UnitTable ut;
  rc = fill_units(ut, h_m, L, rb, h_units, nunits);
  if (rc) return rc;
  BsplineSpec bs;
  rc = fill_bspline(bs, ngroups, h_order, h_start, h_comps, h_scale, d);
  if (rc) return rc;
  const int tail = d - t1;
  if ((int64_t)rb * tail > SFFT_ANCHOR_MAX) return E_2BIG;
  AnchorTable at;
  at.rb = rb;
  at.tail = tail;
  for (int i = 0; i < rb * tail; ++i) at.a[i] = h_anchor[i];
  return launch_sample_bspline(ut, lt, bs, at, (const double2*)d_chirp, (double2*)d_buf, P,
                               mulmod_fast(h_m, L), apply_chirp != 0, num_sms_current(),
                               S(stream));
}

int sfft_finish_samples(const int64_t* h_m, int L, int rb, const double* d_chirp, double* d_buf,
                        int64_t P, const double* d_noise, int64_t nstride, const double* d_sigma,
                        const int32_t* h_units, int nunits, void* stream) {
  UnitTable ut;
  int rc = fill_units(ut, h_m, L, rb, h_units, nunits);
  if (rc) return rc;
  return launch_finish_samples(ut, (const double2*)d_chirp, (double2*)d_buf, P,
                               (const double2*)d_noise, nstride, d_sigma, num_sms_current(),
                               S(stream));
}

int sfft_finish_devnoise(const int64_t* h_m, int L, int rb, const double* d_chirp, double* d_buf,
                         int64_t P, const double* d_norm2, double rel, double sigma, uint64_t seed,
                         uint64_t call_base, int apply_chirp, const int32_t* h_units, int nunits,
                         void* stream) {
  UnitTable ut;
  int rc = fill_units(ut, h_m, L, rb, h_units, nunits);
  if (rc) return rc;
  return launch_finish_devnoise(ut, (const double2*)d_chirp, (double2*)d_buf, P, d_norm2, rel, sigma,
                                seed, call_base, apply_chirp != 0, num_sms_current(), S(stream));
}

int sfft_unit_norm2(const int64_t* h_m, int L, int rb, const double* d_buf, int64_t P,
                    double* d_out, const int32_t* h_units, int nunits, void* stream) {
  UnitTable ut;
  int rc = fill_units(ut, h_m, L, rb, h_units, nunits);
  if (rc) return rc;
  return launch_unit_norm2(ut, (const double2*)d_buf, P, d_out, num_sms_current(), S(stream));
}

int sfft_lattice_nodes(const int64_t* h_m, const int32_t* h_z, int L, int t1, int l, int d,
                       const double* h_anchor_tail, double* d_pts, void* stream) {
  if (l < 0 || l >= L || t1 < 1 || t1 > d || d > SFFT_DMAX) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, h_m, h_z, L, t1);
  if (rc) return rc;
  AnchorTable at;
  at.rb = 1;
  at.tail = d - t1;
  for (int i = 0; i < d - t1; ++i) at.a[i] = h_anchor_tail[i];
  return launch_lattice_nodes(lt, l, d, at, 0, d_pts, mulmod_fast(h_m, L), S(stream));
}

int sfft_gather_select(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax, const int64_t* h_m,
                       const int32_t* h_z, int L, const uint64_t* d_masks, const double* d_buf,
                       int64_t P, int rb, int it0, double delta, double* d_coef, uint8_t* d_keep,
                       int32_t* d_counts, void* stream) {
  if (n < 0 || rb < 1 || rb > 8 || it0 < 0) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, h_m, h_z, L, t1);
  if (rc) return rc;
  return launch_gather(d_freqs, n, lt, d_masks, (const double2*)d_buf, P, rb, it0, delta,
                       (double2*)d_coef, d_keep, d_counts, fast_i32(lt, t1, kmax, h_m, L),
                       num_sms_current(), S(stream));
}

int sfft_gather_units(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax, const int64_t* h_m,
                      const int32_t* h_z, int L, const uint64_t* d_masks, const double* d_buf,
                      int64_t P, int rb, const int32_t* h_units, int nunits, double* d_out,
                      void* stream) {
  if (n < 0 || !h_units) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, h_m, h_z, L, t1);
  if (rc) return rc;
  UnitTable ut;
  rc = fill_units(ut, h_m, L, rb, h_units, nunits);
  if (rc) return rc;
  return launch_gather_units(d_freqs, n, lt, d_masks, (const double2*)d_buf, P, ut, (double2*)d_out,
                             fast_i32(lt, t1, kmax, h_m, L), num_sms_current(), S(stream));
}

int64_t sfft_mask_tiles_len(int64_t n, int L) { return ((n + 255) / 256) * (int64_t)L; }

int sfft_mask_tiles(const uint64_t* d_masks, int64_t n, int L, int32_t* d_tc, int32_t* d_toff, int64_t ts, int W,
                    int32_t* d_sc, void* stream) {
  if (n < 0) return E_INVAL;
  return launch_mask_tiles(d_masks, n, L, d_tc, d_toff, ts, W, d_sc, num_sms_current(), S(stream));
}

int sfft_pack_units(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax, const int64_t* h_m, const int32_t* h_z,
                    int L, const uint64_t* d_masks, const double* d_buf, int64_t P, int rb, const int32_t* h_units,
                    int nunits, const int32_t* d_toff, int64_t ts, const int64_t* d_soff, double* d_send,
                    void* stream) {
  if (n < 0 || !h_units || ts < 1) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, h_m, h_z, L, t1);
  if (rc) return rc;
  UnitTable ut;
  rc = fill_units(ut, h_m, L, rb, h_units, nunits);
  if (rc) return rc;
  return launch_pack_units(d_freqs, n, lt, d_masks, (const double2*)d_buf, P, ut, d_toff, ts, d_soff,
                           (double2*)d_send, fast_i32(lt, t1, kmax, h_m, L), num_sms_current(), S(stream));
}

int sfft_combine_slice(int64_t n, int L, const uint64_t* d_masks, const int32_t* d_toff, int64_t ts, int q,
                       const double* d_recv, const int64_t* d_roff, int rb, double delta, double* d_coef_s,
                       uint8_t* d_keep_s, int32_t* d_counts, void* stream) {
  if (n < 0 || L < 1 || L > SFFT_LMAX || rb < 1 || rb > 8 || q < 0 || ts < 1) return E_INVAL;
  return launch_combine_slice(n, L, d_masks, d_toff, ts, q, (const double2*)d_recv, d_roff, rb, delta,
                              (double2*)d_coef_s, d_keep_s, d_counts, num_sms_current(), S(stream));
}

int sfft_unshard_rows(const void* d_in, int elem, int W, int rb, int64_t S_, int64_t n, int it0, void* d_out,
                      void* stream) {
  if (W < 1 || rb < 1 || S_ < 0 || n < 0 || it0 < 0) return E_INVAL;
  return launch_unshard(d_in, elem, W, rb, S_, n, it0, d_out, num_sms_current(), S(stream));
}

int sfft_combine_units(int64_t n, int L, const uint64_t* d_masks, const double* d_vals,
                       const int32_t* h_rows, int r_total, int rb, int it0, double delta,
                       double* d_coef, uint8_t* d_keep, int32_t* d_counts, void* stream) {
  if (n < 0 || L < 1 || L > SFFT_LMAX || rb < 1 || rb > 8 || it0 < 0 || it0 + rb > r_total)
    return E_INVAL;
  if ((int64_t)r_total * L > SFFT_UMAX) return E_2BIG;
  RowMap rm;
  for (int u = 0; u < r_total * L; ++u) rm.row[u] = h_rows[u];
  return launch_combine_units(n, L, d_masks, (const double2*)d_vals, rm, rb, it0, delta,
                              (double2*)d_coef, d_keep, d_counts, num_sms_current(), S(stream));
}

int64_t sfft_select_scratch_bytes(int64_t n) { return select_scratch_bytes(n); }

int sfft_select_cap(const double* d_coef, uint8_t* d_keep, int64_t n, int cap, uint8_t* d_scratch,
                    void* stream) {
  if (n < 0 || cap < 0) return E_INVAL;
  return launch_select_cap((const double2*)d_coef, d_keep, n, cap, d_scratch, num_sms_current(),
                           S(stream));
}

int64_t sfft_select_rows_scratch_bytes(int nrows) { return select_rows_scratch_bytes(nrows); }

int sfft_select_cap_rows(const double* d_coef, uint8_t* d_keep, int64_t n, const int32_t* h_rows, int nrows,
                         int cap, int32_t* d_counts, uint8_t* d_scratch, void* stream) {
  if (n < 0 || cap < 0 || nrows < 0 || nrows > 64) return E_INVAL;
  return launch_select_cap_rows((const double2*)d_coef, d_keep, n, h_rows, nrows, cap, d_counts, d_scratch,
                                num_sms_current(), S(stream));
}

int64_t sfft_scan_scratch_len(int64_t n) { return scan_scratch_len(n); }

int sfft_flag_indices(const uint8_t* d_flags, int64_t n, int nrows, int32_t* d_idx,
                      int32_t* d_total, int32_t* d_scratch, void* stream) {
  if (n < 0 || n > 0x7fffffffLL || nrows < 1) return E_INVAL;
  return launch_flag_indices(d_flags, n, nrows, d_idx, d_total, d_scratch, S(stream));
}

int sfft_zero_async(void* dst, int64_t nbytes, void* stream) {
  if (nbytes < 0 || (nbytes > 0 && !dst)) return E_INVAL;
  if (nbytes == 0) return 0;
  return (int)cudaMemsetAsync(dst, 0, (size_t)nbytes, S(stream));
}

int sfft_masks_covered(const uint64_t* d_masks, int64_t n, uint8_t* d_out, void* stream) {
  if (n < 0 || (n > 0 && (!d_masks || !d_out)) || ((uintptr_t)d_out & 7)) return E_INVAL;
  return launch_masks_covered(d_masks, n, d_out, num_sms_current(), S(stream));
}

int sfft_gather_rows(const int32_t* d_in, int64_t n_in, int ncomp, const int32_t* d_idx,
                     const int32_t* d_count, int64_t cap_rows, int32_t* d_out, int64_t out_stride,
                     const double* d_cin, double* d_cout, void* stream) {
  return launch_gather_rows(d_in, n_in, ncomp, d_idx, d_count, cap_rows, d_out, out_stride,
                            (const double2*)d_cin, (double2*)d_cout, num_sms_current(), S(stream));
}

int sfft_candidate_product(const int32_t* d_prefix, int64_t np, int t, const int32_t* d_comp,
                           int64_t nc, int32_t* d_out, void* stream) {
  if (np < 0 || nc < 0 || t < 0) return E_INVAL;
  return launch_product(d_prefix, np, t, d_comp, nc, d_out, num_sms_current(), S(stream));
}

int sfft_residues(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax, const int64_t* h_m,
                  const int32_t* h_z, int L, int64_t* d_out, void* stream) {
  if (n < 0 || t1 < 1) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, h_m, h_z, L, t1);
  if (rc) return rc;
  return launch_residues(d_freqs, n, lt, d_out, fast_i32(lt, t1, kmax, h_m, L), num_sms_current(),
                         S(stream));
}

int sfft_line_sample_poly(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int t,
                          int K, const double* h_anchors, int r, double* d_values, void* stream) {
  if ((int64_t)r * d > 2048 || t < 0 || t >= d) return E_2BIG;
  LineAnchors la;
  for (int i = 0; i < r * d; ++i) la.a[i] = h_anchors[i];
  return launch_line_sample_poly(d_hfreqs, (const double2*)d_hcoef, s, d, t, K, la, r,
                                 (double2*)d_values, S(stream));
}

int sfft_line_sample_poly_all(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int K,
                              const double* h_anchors, int r, double* d_values, void* stream) {
  if (d < 1 || r < 1 || (int64_t)d * r * d > 2048) return E_2BIG;
  LineAnchors la;
  for (int i = 0; i < d * r * d; ++i) la.a[i] = h_anchors[i];
  return launch_line_sample_poly_all(d_hfreqs, (const double2*)d_hcoef, s, d, K, la, r, (double2*)d_values,
                                     S(stream));
}

int sfft_line_select(const double* d_values, int r, int K, int64_t lo, int cap, double delta,
                     double* d_coefs, uint8_t* d_keep, void* stream) {
  return launch_line_select((const double2*)d_values, r, K, lo, cap, delta, (double2*)d_coefs,
                            d_keep, S(stream));
}

int sfft_line_bins(const double* d_spectra, int64_t P, int r, int K, int64_t lo, double delta,
                   double* d_coefs, uint8_t* d_keep, int32_t* d_counts, void* stream) {
  return launch_line_bins((const double2*)d_spectra, P, r, K, lo, delta, (double2*)d_coefs, d_keep, d_counts,
                          num_sms_current(), S(stream));
}

int sfft_eval_poly_points(const double* d_pts, int64_t n, int d, const int32_t* d_hfreqs,
                          const double* d_hcoef, int s, double* d_out, void* stream) {
  if (n < 0 || d < 1 || s < 0) return E_INVAL;
  return launch_eval_poly_points(d_pts, n, d, d_hfreqs, (const double2*)d_hcoef, s,
                                 (double2*)d_out, S(stream));
}

int sfft_line_points(const double* d_anchors, int d, int r, int K, double* d_pts, void* stream) {
  if (d < 1 || r < 1 || K < 1) return E_INVAL;
  return launch_line_points(d_anchors, d, r, K, d_pts, num_sms_current(), S(stream));
}

int sfft_eval_bspline_points(const double* d_pts, int64_t n, int d, int ngroups,
                             const int32_t* h_order, const int32_t* h_start,
                             const int32_t* h_comps, const double* h_scale, double* d_out,
                             void* stream) {
  BsplineSpec bs;
  int rc = fill_bspline(bs, ngroups, h_order, h_start, h_comps, h_scale, d);
  if (rc) return rc;
  return launch_eval_bspline_points(d_pts, n, bs, (double2*)d_out, num_sms_current(), S(stream));
}

int sfft_add_noise(double* d_x, const double* d_noise, int64_t n, double scale, void* stream) {
  if (n < 0) return E_INVAL;
  return launch_add_noise((double2*)d_x, (const double2*)d_noise, n, scale, num_sms_current(),
                          S(stream));
}

int sfft_cbc_scan(const int64_t* d_prefix_res, const int32_t* d_col, int64_t n, int64_t m, int64_t z0,
                  int Z, uint32_t* d_bits, int64_t words, int32_t* d_dup, void* stream) {
  if (n < 0 || m < 1 || m > 2147483647LL || Z < 0 || words < (m + 31) / 32) return E_INVAL;
  return launch_cbc_scan(d_prefix_res, d_col, n, m, z0, Z, d_bits, words, d_dup, num_sms_current(),
                         S(stream));
}

int sfft_prefix_flags(const int32_t* d_freqs, int64_t n, int t1, uint8_t* d_flags, void* stream) {
  if (n < 0 || t1 < 1) return E_INVAL;
  return launch_prefix_flags(d_freqs, n, t1, d_flags, num_sms_current(), S(stream));
}

int sfft_scatter_residues(const int32_t* d_freqs, int64_t n, int t1, int64_t m, const int32_t* h_z,
                          const double* d_coef, double* d_acc, void* stream) {
  if (n < 0 || t1 < 1) return E_INVAL;
  LatTable lt;
  int rc = fill_lat(lt, &m, h_z, 1, t1);
  if (rc) return rc;
  return launch_scatter_residues(d_freqs, n, lt, (const double2*)d_coef, (double2*)d_acc,
                                 num_sms_current(), S(stream));
}

int sfft_pack_rows(const int64_t* d_rows, int64_t n, int d, int32_t* d_out, int32_t* d_minmax,
                   void* stream) {
  if (n < 0) return E_INVAL;
  return launch_pack_rows(d_rows, n, d, d_out, d_minmax, num_sms_current(), S(stream));
}

int sfft_cscale(double* d_x, int64_t n, double scale, int conj, void* stream) {
  return launch_cscale((double2*)d_x, n, scale, conj, num_sms_current(), S(stream));
}

int sfft_fp64_peak(double* d_out, int iters, int blocks, void* stream) {
  return launch_fp64_peak(d_out, iters, blocks, S(stream));
}

int sfft_fp64_mma_peak(double* d_out, int iters, int blocks, void* stream) {
  return launch_fp64_mma_peak(d_out, iters, blocks, S(stream));
}

int sfft_l2_random_peak(uint32_t* d_bits, int64_t words, int blocks, int per_thread, int mode, void* stream) {
  if (words < 1 || words > 0x7fffffffLL || blocks < 1 || per_thread < 1 || mode < 0 || mode > 2) return E_INVAL;
  return launch_l2_random_peak(d_bits, (uint32_t)words, blocks, per_thread, mode, S(stream));
}

}  // extern "C"
