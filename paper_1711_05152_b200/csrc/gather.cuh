#pragma once
#include "plan.cuh"

namespace sfft {

// words: the two bitmaps' words of lattices [0, nlat) (their layout);
// capacity: the scratch's words (the 32-bit counter variant when they fit)
int launch_alias(const int32_t* freqs, int64_t n, const LatTable& lt, int l0, uint32_t* bits,
                 int64_t words, int64_t capacity, uint64_t* masks, int32_t* stats, bool fast, int num_sms,
                 cudaStream_t st);
bool alias_counters_for(const int64_t* m, int L);
int64_t alias_scratch_words(const LatTable& lt);
int launch_gather(const int32_t* freqs, int64_t n, const LatTable& lt, const uint64_t* masks,
                  const double2* buf, int64_t ustride, int rb, int it0, double delta, double2* coef,
                  uint8_t* keep, int32_t* counts, bool fast, int num_sms, cudaStream_t st);
int launch_gather_units(const int32_t* freqs, int64_t n, const LatTable& lt, const uint64_t* masks,
                        const double2* buf, int64_t ustride, const UnitTable& ut, double2* out,
                        bool fast, int num_sms, cudaStream_t st);
int launch_combine_units(int64_t n, int L, const uint64_t* masks, const double2* vals,
                         const RowMap& rm, int rb, int it0, double delta, double2* coef,
                         uint8_t* keep, int32_t* counts, int num_sms, cudaStream_t st);
int64_t scan_scratch_len(int64_t n);
int launch_flag_indices(const uint8_t* flags, int64_t n, int nrows, int32_t* idx_out,
                        int32_t* total, int32_t* scratch, cudaStream_t st);
int launch_masks_covered(const uint64_t* masks, int64_t n, uint8_t* out, int num_sms, cudaStream_t st);
int launch_gather_rows(const int32_t* in, int64_t n_in, int ncomp, const int32_t* idx,
                       const int32_t* count, int64_t cap_rows, int32_t* out, int64_t out_stride,
                       const double2* cin, double2* cout, int num_sms, cudaStream_t st);
int64_t select_scratch_bytes(int64_t n);
int64_t select_rows_scratch_bytes(int nrows);
int launch_select_cap_rows(const double2* coef, uint8_t* keep, int64_t n, const int32_t* h_rows, int nrows,
                           int cap, int32_t* counts, uint8_t* scratch, int num_sms, cudaStream_t st);
int launch_select_cap(const double2* coef, uint8_t* keep, int64_t n, int cap, uint8_t* scratch,
                      int num_sms, cudaStream_t st);
int launch_product(const int32_t* pref, int64_t np, int t, const int32_t* comp, int64_t nc,
                   int32_t* out, int num_sms, cudaStream_t st);
int launch_residues(const int32_t* freqs, int64_t n, const LatTable& lt, int64_t* out, bool fast,
                    int num_sms, cudaStream_t st);
int launch_pack_rows(const int64_t* rows, int64_t n, int d, int32_t* out, int32_t* minmax,
                     int num_sms, cudaStream_t st);
int launch_cscale(double2* x, int64_t n, double scale, int conj, int num_sms, cudaStream_t st);

}  // namespace sfft
