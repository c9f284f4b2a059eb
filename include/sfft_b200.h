/*
 * sfft_b200.h — C ABI of the B200 multiple-rank-1-lattice (MR1L) hot path.
 *
 * The reference (arXiv 1711.05152 package `sfft`, /root/reference/pkg/src/sfft)
 * is pure Python; it has no native boundary.  These entry points replace the
 * internal seams of its MR1L reconstruction step one-for-one, and
 * are bound from Python with ctypes by paper_1711_05152_b200/_native.py.
 *
 * Conventions
 *   - d_* arguments are DEVICE pointers owned by the caller; h_* are HOST
 *     pointers to small metadata (copied into kernel parameters, never
 *     retained).  No call allocates device memory; scratch is caller-provided.
 *   - Every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and returns 0 on success, a cudaError_t value (> 0) on a
 *     CUDA error, or a negative errno-style code on an argument error.
 *     sfft_error_string() names the code.
 *   - Frequency sets are component-major int32: freqs[c * n + i] is component c
 *     of candidate i (|k_c| <= 2^31 - 1, lattice.py:36-38).  Candidate sets are
 *     kept lexicographically sorted (lattice.py:63-77).
 *   - Complex arrays are interleaved complex128 (double re, im).
 *   - Lattice metadata: h_m[l] = M_l (1 <= M_l <= 2^31 - 1), h_z[l * t1 + c]
 *     = z_l[c] in [0, M_l) (lattice.py:284-294).  One "unit" is one
 *     (iteration i, lattice l) pair, numbered u = i * L + l; unit u owns the
 *     transform buffer d_buf + 2 * u * P doubles.
 *   - Thread-safe across distinct streams / devices; one host thread per GPU.
 */
#ifndef SFFT_B200_H
#define SFFT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ABI history: 4 = sfft_copy_async, sfft_zero_async, sfft_masks_covered,
 * sfft_line_points and sfft_line_sample_poly_all added (no signature changed).  3 = anchor tables of the sampling entries limited to
 * rb * (d - t1) <= 512 doubles (2 allowed 1024; larger now returns -7, E_2BIG,
 * for every d), sfft_unit_norm2 deterministic (cluster reduction). */
#define SFFT_B200_ABI_VERSION 4

int sfft_abi_version(void);
/* kernels launched by this library since load (all devices, all streams) */
long long sfft_launch_count(void);
/* CUDA-event timing of kernel classes on their launching stream:
 * 0 = polynomial sampling GEMM (K1), 1 = Bluestein FFT passes (K2),
 * 2 = alias histogram + masks (K3), 3 = gather/average/threshold (K4).
 * enable(1) clears the record; collect() synchronises and returns the summed
 * device time and launch count of one class since the last collect. */
int sfft_profile_enable(int on);
int sfft_profile_collect(int cls, double* total_ms, int* count);
const char* sfft_error_string(int code);
/* number of SMs and compute capability of the current device */
int sfft_device_info(int* num_sms, int* cc_major, int* cc_minor);
/* cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDefault, stream): the engine's
 * read-backs of small results into pinned host buffers (host page-locked
 * memory for an asynchronous copy), without a framework's stream switch */
int sfft_copy_async(void* dst, const void* src, int64_t nbytes, void* stream);
/* cudaMemsetAsync(dst, 0, nbytes, stream): zeroed counters of the engine */
int sfft_zero_async(void* dst, int64_t nbytes, void* stream);
/* d_out[i] = (d_masks[i] != 0) for i < n: a scheme's coverage of its target
 * set (MultipleRank1Lattice coverage, lattice.py) as bytes; d_out 8-byte
 * aligned. */
int sfft_masks_covered(const uint64_t* d_masks, int64_t n, uint8_t* d_out, void* stream);

/* ---- K3: alias histogram, masks, coverage --------------------------------
 * Replaces construct.py:139-143 (_alias_free_mask) evaluated for every prime
 * of one attempt of build_multiple_lattice (construct.py:146-182), with
 * residues as lattice.py:511-517.  masks[i] bit l = candidate i is alias-free
 * on lattice l.  stats[0] = max_i (index of the lowest set bit + 1) (the
 * early-exit lattice count when every mask is nonzero), stats[1] = number of
 * candidates with an empty mask.  kmax bounds |k_c| (selects exact fast
 * arithmetic when d*kmax*M < 2^52).  L <= 64, L * t1 <= 4096, t1 <= 64. */
int64_t sfft_alias_scratch_words(const int64_t* h_m, int L);
int sfft_alias_masks(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax,
                     const int64_t* h_m, const int32_t* h_z, int L,
                     uint32_t* d_scratch, int64_t scratch_words,
                     uint64_t* d_masks, int32_t* d_stats, void* stream);
/* The same for lattices [l0, l1) only (h_m, h_z cover lattices [0, l1);
 * scratch sized by sfft_alias_scratch_words(h_m, l1)).  l0 > 0 adds their bits
 * to masks holding lattices [0, l0) from an earlier call, and the stats then
 * cover all l1 lattices: the per-prime early-exit loop of construct.py:173-181
 * evaluated a chunk of primes at a time. */
int sfft_alias_masks_range(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax,
                           const int64_t* h_m, const int32_t* h_z, int l0, int l1,
                           uint32_t* d_scratch, int64_t scratch_words,
                           uint64_t* d_masks, int32_t* d_stats, void* stream);

/* ---- per-lattice tables ----------------------------------------------------
 * tw[off_l + n] = e^{+2 pi i n / M_l}, chirp[off_l + n] = e^{-pi i (n^2 mod 2M_l)/M_l},
 * off_l = sum_{l' < l} M_l' (both arrays hold sum_l M_l complex values). */
int sfft_lattice_tables(const int64_t* h_m, int L, double* d_tw, double* d_chirp, void* stream);

/* ---- K2: Bluestein prime-length DFT (transform.py:50-64, scipy.fft.fft) -----
 * Cyclic convolution length P >= 2 * max M_l - 1: sfft_fft_size(max M_l)
 * returns the library's choice (a power of two up to 2048; above that
 * P = f * 2^a * 2048 with f in {1, 3, 5, 7, 9, 25}, within 1.33x of
 * 2 M - 1; powers of two 2^23, 2^24 for the largest sizes; -1 above 2^24;
 * SFFT_B200_FFT_POW2=1 restricts it to powers of two).  sfft_fft_tables
 * fills the FFT twiddle tables (sfft_fft_table_len(P) complex values, -1 for
 * an unsupported P); sfft_bluestein_bhat builds the transformed Bluestein
 * kernel of each lattice (L * P complex); sfft_bluestein transforms `nunits`
 * pre-chirped buffers in place and leaves the unnormalised DFT X_k (k < M of
 * the unit's lattice) in d_buf. */
int64_t sfft_fft_size(int64_t m_max);
int64_t sfft_fft_table_len(int64_t P);
int sfft_fft_tables(int64_t P, double* d_ftab, void* stream);
int sfft_bluestein_bhat(const int64_t* h_m, int L, int64_t P, const double* d_ftab,
                        const double* d_chirp, double* d_bhat, void* stream);
int sfft_bluestein(const int64_t* h_m, int L, int rb, int64_t P, const double* d_ftab,
                   const double* d_bhat, const double* d_chirp, double* d_buf,
                   const int32_t* h_units, int nunits, void* stream);

/* Unit lists: functions taking (h_units, nunits) process the explicit units
 * h_units[j] = it * L + l (it < rb), unit j in buffer slot j; h_units = NULL
 * means all rb * L units in order. */

/* ---- K1: sampling at lattice nodes ----------------------------------------
 * Sparse polynomial oracle (testbed.py:116-127) on the nodes of
 * _invert_candidates (detect.py:290-299): unit u = i*L + l gets
 * x_n * chirp_l[n] (n < M_l) in its buffer, x_n = p(node n of lattice l with
 * anchor tail i).  Terms: d_hfreqs component-major (d x s int32), d_hcoef s
 * complex.  h_anchor: rb x (d - t1) doubles, rb * (d - t1) <= 512 (else
 * -7).  Scratch: d_cprime rb*s complex,
 * d_rres and d_rj L*s int32 each, d_partial partial_len complex (term-slice
 * partial sums; sfft_sample_poly_scratch() gives the size for the best
 * split, a smaller buffer selects a smaller split, 0 disables it).
 * apply_chirp = 0 leaves the raw samples. */
int64_t sfft_sample_poly_scratch(const int64_t* h_m, int L, int rb, int s, const int32_t* h_units,
                                 int nunits);
int sfft_sample_poly(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int t1,
                     const int64_t* h_m, const int32_t* h_z, int L,
                     const double* h_anchor, int rb,
                     double* d_cprime, int32_t* d_rres, int32_t* d_rj,
                     const double* d_tw, const double* d_chirp,
                     double* d_buf, int64_t P, int apply_chirp,
                     double* d_partial, int64_t partial_len,
                     const int32_t* h_units, int nunits, void* stream);
/* sfft_sample_poly split in its two phases: _prepare (anchor-rotated
 * coefficients c' for rb iterations, residues r_h and r_h J1 for L lattices;
 * depends on the sizes and vectors only, so it can run for all L_max
 * lattices while the alias kernel decides L) and _run (everything else, for
 * the first L lattices of the prepared set, same arguments as
 * sfft_sample_poly). */
int sfft_sample_poly_prepare(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int t1,
                             const int64_t* h_m, const int32_t* h_z, int L, const double* h_anchor, int rb,
                             double* d_cprime, int32_t* d_rres, int32_t* d_rj, const double* d_tw,
                             double* d_scratch, int64_t scratch_len, int* h_panels_built, void* stream);
/* d_tw / d_scratch (nullable): also build the B panels of the tensor-core
 * kernel (they depend on the lattices only) at the start of the scratch when
 * it is large enough; *h_panels_built (nullable) reports whether they were
 * queued, and sfft_sample_poly_run(panels_ready = 1) then skips them. */
int sfft_sample_poly_run(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int t1,
                         const int64_t* h_m, const int32_t* h_z, int L, const double* h_anchor, int rb,
                         double* d_cprime, int32_t* d_rres, int32_t* d_rj, const double* d_tw,
                         const double* d_chirp, double* d_buf, int64_t P, int apply_chirp,
                         double* d_partial, int64_t partial_len, const int32_t* h_units, int nunits,
                         int panels_ready, void* stream);
/* B-spline oracle (testbed.py:198-244): ngroups tensor-product terms; group g
 * has spline order h_order[g] (<= 8), scale h_scale[g] = C_m * m, and the
 * component slots h_comps[h_start[g] .. h_start[g+1]). */
int sfft_sample_bspline(int ngroups, const int32_t* h_order, const int32_t* h_start,
                        const int32_t* h_comps, const double* h_scale, int d, int t1,
                        const int64_t* h_m, const int32_t* h_z, int L,
                        const double* h_anchor, int rb, const double* d_chirp,
                        double* d_buf, int64_t P, int apply_chirp,
                        const int32_t* h_units, int nunits, void* stream);
/* Host-callback / noisy oracles: d_buf holds raw samples; adds
 * d_sigma[u] * d_noise[u * nstride + n] when d_noise != NULL (NoisyOracle,
 * testbed.py:100-106), then applies the pre-chirp. */
int sfft_finish_samples(const int64_t* h_m, int L, int rb, const double* d_chirp,
                        double* d_buf, int64_t P, const double* d_noise, int64_t nstride,
                        const double* d_sigma, const int32_t* h_units, int nunits, void* stream);
/* Device-generated noise (statistically equivalent to NoisyOracle; realisation
 * from Philox4x32-10 keyed by seed, counter (n, oracle-call index), so it is
 * reproducible and independent of launch splits / GPU counts): unit u (global
 * id g = it * L + l) is oracle call call_base + g; its samples get
 * s_u * (N(0,1) + i N(0,1)) with s_u = sigma / sqrt(2), or, when d_norm2 is
 * given, rel * sqrt(d_norm2[u] / M_l) / sqrt(2); then the optional pre-chirp. */
int sfft_finish_devnoise(const int64_t* h_m, int L, int rb, const double* d_chirp, double* d_buf,
                         int64_t P, const double* d_norm2, double rel, double sigma, uint64_t seed,
                         uint64_t call_base, int apply_chirp, const int32_t* h_units, int nunits,
                         void* stream);
/* sum_n |x_n|^2 per unit over n < M (relative-SNR noise calibration). */
int sfft_unit_norm2(const int64_t* h_m, int L, int rb, const double* d_buf, int64_t P,
                    double* d_out, const int32_t* h_units, int nunits, void* stream);
/* Node coordinates of lattice l (lattice.py:505-508 + anchor tail,
 * detect.py:294-297): d_pts is M_l x d row-major float64. */
int sfft_lattice_nodes(const int64_t* h_m, const int32_t* h_z, int L, int t1, int l, int d,
                       const double* h_anchor_tail, double* d_pts, void* stream);

/* ---- K4: gather + average + threshold (transform.py:99-127, detect.py:197-204)
 * For iterations it0 .. it0+rb-1 (rb <= 8) of the step: coef[(it0+i)*n + k] =
 * average over lattices l < L with mask bit l of X_{i,l}[k.z_l mod M_l] / M_l;
 * keep = |coef| >= delta (0 for uncovered k); counts[it0+i] += #kept. */
int sfft_gather_select(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax,
                       const int64_t* h_m, const int32_t* h_z, int L,
                       const uint64_t* d_masks, const double* d_buf, int64_t P,
                       int rb, int it0, double delta,
                       double* d_coef, uint8_t* d_keep, int32_t* d_counts, void* stream);
/* Sharded step: per-unit dense rows of alias-free bins (out[j*n + k] =
 * X_j[res] / M, 0 where lattice of unit j is not alias-free for k), and their
 * lattice-ordered combination after an all-gather (h_rows[i*L + l] = row of
 * unit (i, l) in d_vals), bit-identical to sfft_gather_select. */
int sfft_gather_units(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax, const int64_t* h_m,
                      const int32_t* h_z, int L, const uint64_t* d_masks, const double* d_buf,
                      int64_t P, int rb, const int32_t* h_units, int nunits, double* d_out,
                      void* stream);
/* ---- sharded step, sliced exchange (replaces the dense-row
 * all-gather of sfft_gather_units / sfft_combine_units, which remain).
 * Candidates are cut into W slices of ts tiles of 256 candidates.
 * sfft_mask_tiles: per-tile popcounts of every mask bit (d_tc, sized
 * sfft_mask_tiles_len), their exclusive scan along the tiles d_toff
 * ((ntiles + 1) x L int32) and the slice totals d_sc (W x L int32).
 * sfft_pack_units: for the listed own units (slot j = buffer slot j, as
 * sfft_gather_units) write X_j[k.z_l mod M_l] * (1/M_l) of every candidate k
 * with mask bit l set, slice-major: slice q of slot j starts at
 * d_soff[q * nunits + j] (complex elements of d_send), candidate order.
 * sfft_combine_slice: slice q's candidates from the received packs (unit
 * u = i * L + l of the chunk at d_roff[u]): lattice-order average, delta
 * threshold -> d_coef_s / d_keep_s ([rb][ts * 256]), survivors into d_counts
 * (rb, zeroed first).  sfft_unshard_rows: [W][rb][S] -> rows it0.. of
 * [r][n] (elem = 1: keep flags, 16: coefficients). */
int64_t sfft_mask_tiles_len(int64_t n, int L);
int sfft_mask_tiles(const uint64_t* d_masks, int64_t n, int L, int32_t* d_tc, int32_t* d_toff, int64_t ts, int W,
                    int32_t* d_sc, void* stream);
int sfft_pack_units(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax, const int64_t* h_m, const int32_t* h_z,
                    int L, const uint64_t* d_masks, const double* d_buf, int64_t P, int rb, const int32_t* h_units,
                    int nunits, const int32_t* d_toff, int64_t ts, const int64_t* d_soff, double* d_send,
                    void* stream);
int sfft_combine_slice(int64_t n, int L, const uint64_t* d_masks, const int32_t* d_toff, int64_t ts, int q,
                       const double* d_recv, const int64_t* d_roff, int rb, double delta, double* d_coef_s,
                       uint8_t* d_keep_s, int32_t* d_counts, void* stream);
int sfft_unshard_rows(const void* d_in, int elem, int W, int rb, int64_t S, int64_t n, int it0, void* d_out,
                      void* stream);
int sfft_combine_units(int64_t n, int L, const uint64_t* d_masks, const double* d_vals,
                       const int32_t* h_rows, int r_total, int rb, int it0, double delta,
                       double* d_coef, uint8_t* d_keep, int32_t* d_counts, void* stream);
/* cap selection of one iteration (detect.py:205-211) */
int64_t sfft_select_scratch_bytes(int64_t n);
int sfft_select_cap(const double* d_coef, uint8_t* d_keep, int64_t n, int cap,
                    uint8_t* d_scratch, void* stream);
/* the same cap selection for `nrows` iterations at once: rows h_rows[i] of
 * d_coef (r, n, 2) / d_keep (r, n); scratch = sfft_select_rows_scratch_bytes.
 * d_counts (nullable, int32 per row): when given, a row is capped only if its
 * survivor count exceeds `cap` (decided on the device, count set to cap), so
 * the caller needs no host read-back of the counts. */
int64_t sfft_select_rows_scratch_bytes(int nrows);
int sfft_select_cap_rows(const double* d_coef, uint8_t* d_keep, int64_t n, const int32_t* h_rows,
                         int nrows, int cap, int32_t* d_counts, uint8_t* d_scratch, void* stream);

/* ---- compaction / sets (detect.py:257-260, 367-371, 412; lattice.py:97-109) */
int64_t sfft_scan_scratch_len(int64_t n);
/* ascending indices i with OR_r flags[r*n + i] != 0; *d_total = count */
int sfft_flag_indices(const uint8_t* d_flags, int64_t n, int nrows, int32_t* d_idx,
                      int32_t* d_total, int32_t* d_scratch, void* stream);
int sfft_gather_rows(const int32_t* d_in, int64_t n_in, int ncomp, const int32_t* d_idx,
                     const int32_t* d_count, int64_t cap_rows, int32_t* d_out, int64_t out_stride,
                     const double* d_cin, double* d_cout, void* stream);
int sfft_candidate_product(const int32_t* d_prefix, int64_t np, int t, const int32_t* d_comp,
                           int64_t nc, int32_t* d_out, void* stream);

/* residues k . z_l mod M_l (lattice.py:511-529) of every candidate on every
 * lattice: d_out[l * n + i], int64. */
int sfft_residues(const int32_t* d_freqs, int64_t n, int t1, int64_t kmax, const int64_t* h_m,
                  const int32_t* h_z, int L, int64_t* d_out, void* stream);

/* ---- line detection (detect.py:175-240) ------------------------------------
 * r lines of K points of component t, anchors h_anchors (r x d, r * d <= 2048).
 * sfft_line_select (K <= 1024): DFT, bins, threshold and cap of each line in
 * one CTA.  Longer lines: pre-chirp + sfft_bluestein as for a lattice of size
 * K (one unit per line), then sfft_line_bins maps the spectra (row i at
 * d_spectra + 2 * i * P doubles) to coefficients of k = lo .. lo + K - 1
 * (bin k mod K, times 1/K), threshold flags and per-line survivor counts;
 * the cap is sfft_select_cap_rows with those counts. */
int sfft_line_sample_poly(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int t,
                          int K, const double* h_anchors, int r, double* d_values, void* stream);
/* The r lines of every component t < d in one launch (a centred box: the
 * same K <= 1024 for all components): line g = t * r + i with anchors
 * h_anchors[g * d ...] (d * r * d <= 2048 doubles), values row g; the same
 * samples as d calls of sfft_line_sample_poly. */
int sfft_line_sample_poly_all(const int32_t* d_hfreqs, const double* d_hcoef, int s, int d, int K,
                              const double* h_anchors, int r, double* d_values, void* stream);
int sfft_line_bins(const double* d_spectra, int64_t P, int r, int K, int64_t lo, double delta,
                   double* d_coefs, uint8_t* d_keep, int32_t* d_counts, void* stream);
int sfft_line_select(const double* d_values, int r, int K, int64_t lo, int cap, double delta,
                     double* d_coefs, uint8_t* d_keep, void* stream);

/* ---- oracle evaluation at arbitrary points (testbed.py:60-73, 116-127, 232-244)
 * d_pts: n x d row-major float64 in [0,1)^d; d_out: n complex.  These back the
 * device oracles' __call__ and the line samples of non-polynomial oracles. */
/* The points of r anchored axis lines of every component (K points each):
 * row g K + l (g = t r + i) = d_anchors[g d ...] with component t = g / r set
 * to l / K; d_pts is (d r K) x d row-major (line samples of a black-box
 * oracle at all components' lines, detect.py:175-240). */
int sfft_line_points(const double* d_anchors, int d, int r, int K, double* d_pts, void* stream);
int sfft_eval_poly_points(const double* d_pts, int64_t n, int d, const int32_t* d_hfreqs,
                          const double* d_hcoef, int s, double* d_out, void* stream);
int sfft_eval_bspline_points(const double* d_pts, int64_t n, int d, int ngroups,
                             const int32_t* h_order, const int32_t* h_start,
                             const int32_t* h_comps, const double* h_scale, double* d_out,
                             void* stream);
/* d_x[i] += scale * d_noise[i] (complex; NoisyOracle update, testbed.py:104-106) */
int sfft_add_noise(double* d_x, const double* d_noise, int64_t n, double scale, void* stream);

/* ---- single rank-1 lattice (Algorithm 5; construct.py:212-278, transform.py:67-96)
 * CBC scan: d_dup[j] = 1 iff (prefix_res_i + col_i * (z0 + j)) mod m has a
 * repeated value over i < n (d_bits: Z * words scratch, words >= ceil(m/32)).
 * prefix_flags: first row of every distinct t1-prefix of a sorted set.
 * scatter_residues: acc[k . z mod m] += coef_k (eval_on_lattice). */
int sfft_cbc_scan(const int64_t* d_prefix_res, const int32_t* d_col, int64_t n, int64_t m, int64_t z0,
                  int Z, uint32_t* d_bits, int64_t words, int32_t* d_dup, void* stream);
int sfft_prefix_flags(const int32_t* d_freqs, int64_t n, int t1, uint8_t* d_flags, void* stream);
int sfft_scatter_residues(const int32_t* d_freqs, int64_t n, int t1, int64_t m, const int32_t* h_z,
                          const double* d_coef, double* d_acc, void* stream);

/* ---- utilities ---------------------------------------------------------------- */
/* numpy rows (n x d int64, row-major) -> component-major int32 candidates;
 * d_minmax (2d + 1 int32): per-component min, max, and an out-of-range flag
 * (|k| > 2^31 - 1, lattice.py:36-38). */
int sfft_pack_rows(const int64_t* d_rows, int64_t n, int d, int32_t* d_out, int32_t* d_minmax,
                   void* stream);
int sfft_cscale(double* d_x, int64_t n, double scale, int conj, void* stream);
/* FP64 roofline probe: blocks x 256 threads x iters x 16 DFMA */
int sfft_fp64_peak(double* d_out, int iters, int blocks, void* stream);
/* FP64 tensor-core (DMMA m8n8k4) peak loop: blocks x 256 threads, iters x 16
 * MMAs per warp (512 flop each).  K1's roofline denominator is the larger of
 * this and the DFMA loop above. */
int sfft_fp64_mma_peak(double* d_out, int iters, int blocks, void* stream);
/* K3 roofline probe: blocks x 256 threads x per_thread random 32-bit
 * operations on a bitmap of `words` words (size it like the alias scratch so
 * it is L2-resident): mode 0 atomicOr with the old value used, mode 1 loads,
 * mode 2 atomicAdd with the result unused (RED, the alias counter variant). */
int sfft_l2_random_peak(uint32_t* d_bits, int64_t words, int blocks, int per_thread, int mode, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SFFT_B200_H */
