/*
 * aliaskit_b200.h — C ABI of the B200 alias-table library (libaliaskit_b200.so).
 *
 * This is the drop-in boundary for the reference package `aliaskit`
 * (/root/reference/pkg/src/aliaskit).  The reference dispatches every hot
 * loop through one operator layer — `backend.compile_kernel` plus a
 * `kern = X_nb if using_numba() else X` call site (backend.py:62-73) — and
 * each entry point below replaces one such kernel call site.  Kernels there
 * are pure functions over caller-allocated arrays returning small scalars;
 * the same contract holds here:
 *
 *   - all array arguments are DEVICE pointers allocated by the caller
 *     (wrappers allocate outputs, pack.py:272-273, partition.py:110-113,
 *     sample.py:130); functions marked [host] take host pointers;
 *   - `stream` is a cudaStream_t (may be NULL = legacy default stream); calls
 *     are stream-ordered and asynchronous unless marked [sync];
 *   - scratch comes from a caller workspace sized by a *_workspace_bytes
 *     query; the library never frees caller memory.  Its only state, per
 *     (host thread, device, stream), is a 256-byte device status buffer and
 *     a 256-byte mapped pinned host mailbox for the [sync] entry points that
 *     read back a flag or count (a one-block kernel writes the result into
 *     the mailbox, so a readback never queues behind bulk copies on the copy
 *     engines; both allocated on first use, freed at thread exit); the
 *     device-attribute and kernel-attribute set-up is done once per process;
 *   - every function returns an ak_status; Python wrappers map the codes 1:1
 *     onto the reference exceptions (model.py:32-46, split.py:28-33,
 *     pack.py:26-27, sample.py:40-41, stats.py:17-22).
 *
 * Weight dtype: AK_F32 (float) or AK_F64 (double).  Table rows (device):
 *   AK_F32: struct { float  tw; uint32_t alias; }   8 B, alias 1-based
 *   AK_F64: struct { double tw; uint64_t alias; }  16 B, alias 1-based
 *           (= the ALT1 on-disk row, io.py:21)
 * An alias of 0 marks an unwritten row (pack.py:275).
 */
#ifndef ALIASKIT_B200_H
#define ALIASKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AK_OK = 0,
    AK_ERR_EMPTY_INPUT = 1,           /* model.EmptyInput */
    AK_ERR_INVALID_WEIGHT = 2,        /* model.InvalidWeight (bad index out-param) */
    AK_ERR_SIZE_MISMATCH = 3,         /* model.SizeMismatch */
    AK_ERR_INVALID_SECTION_COUNT = 4, /* split.InvalidSectionCount */
    AK_ERR_UNSORTED_INPUT = 5,        /* split.UnsortedInput */
    AK_ERR_PLAN_INCONSISTENT = 6,     /* pack.PlanInconsistent */
    AK_ERR_INVALID_SECTION_SIZE = 7,  /* sample.InvalidSectionSize */
    AK_ERR_VALUE = 8,                 /* plain ValueError (argument checks) */
    AK_ERR_CUDA = 9,                  /* CUDA runtime failure -> RuntimeError */
    AK_ERR_WORKSPACE = 10,            /* workspace too small -> RuntimeError */
    AK_ERR_INDEX_OUT_OF_RANGE = 11,   /* stats.IndexOutOfRange */
} ak_status;

enum { AK_F32 = 0, AK_F64 = 1 };
/* Sample index dtype: AK_I64 (int64, the reference's dtype, sample.py:116)
 * or AK_I32 (opt-in, tables with n <= 2^31-1: half the output bytes, the
 * same 1-based values) */
enum { AK_I32 = 2, AK_I64 = 3 };
enum { AK_RNG_REFERENCE = 0, /* Philox2x64-10 word 0, bit-exact with rng.py */
       AK_RNG_PHILOX4X32 = 1 /* GPU-native Philox4x32-10, two 53-bit draws per call */ };

/* Library identity and the message of the last AK_ERR_CUDA (thread-local). */
const char *ak_version(void);
const char *ak_last_error(void);
size_t ak_row_bytes(int dtype);

/* ---- rng (rng.py) ------------------------------------------------------- */

/* uniform_block (rng.py:153-164): out[i] = uniform(ctr0+i, stream_id, seed),
 * f64 in [0,1), counters wrap mod 2^64.  Replaces the _fill_uniform_nb call
 * at rng.py:156. */
int ak_fill_uniform(uint64_t seed, uint64_t stream_id, uint64_t ctr0, uint64_t m, double *out,
                    void *stream);
/* Raw Philox2x64-10 words (both lanes) for known-answer tests. */
int ak_philox2x64(const uint64_t *ctr, const uint64_t *strm, const uint64_t *key, uint64_t m,
                  uint64_t *out_w0, uint64_t *out_w1, void *stream);
/* Raw Philox4x32-10 (Random123 constants; the GPU-native RNG mode) for
 * known-answer tests: ctr 4 words and key 2 words per input; out 12 words
 * per input = the generic, inline-key and round-key-table formulations the
 * samplers use (all three must agree).  Not a reference call site: the
 * reference has only Philox2x64-10 (rng.py). */
int ak_philox4x32(const uint32_t *ctr, const uint32_t *key, uint64_t m, uint32_t *out,
                  void *stream);
/* derive_stream (rng.py:167-169) [host]. */
uint64_t ak_derive_stream(uint64_t seed, uint64_t stream_id, uint64_t tag0, uint64_t tag1);

/* ---- make_weight_set (model.py:95-108) ---------------------------------- */

size_t ak_weights_workspace_bytes(uint64_t n);
/* [sync] Validates finite and > 0 (first bad 0-based index -> *bad_index,
 * AK_ERR_INVALID_WEIGHT) and computes the total exactly as np.sum (numpy's
 * pairwise tree over the values upcast to f64) -> *total [host]. */
int ak_weights_validate_total(const void *w, int dtype, uint64_t n, double *total,
                              int64_t *bad_index, void *ws, size_t ws_bytes, void *stream);

/* ---- partition_items (partition.py:106-131) ----------------------------- */

size_t ak_partition_workspace_bytes(uint64_t n);
/* [sync] Stable light (w <= avg) / heavy classification in ascending item
 * order with co-located weights, and exclusive compensated prefix sums.
 * l_idx/h_idx: int64 1-based, capacity n; l_w/h_w: weight dtype, capacity n;
 * lprefix/hprefix: f64, capacity n+1.  Prefixes are double-double exact sums
 * rounded to f64 (the reference's are Neumaier-compensated).  Replaces
 * _classify_kernel_nb / _prefix_kernel_nb (partition.py:109-129). */
int ak_partition(const void *w, int dtype, uint64_t n, double avg, int64_t *l_idx, void *l_w,
                 int64_t *h_idx, void *h_w, double *lprefix, double *hprefix, uint64_t *nl_out,
                 uint64_t *nh_out, void *ws, size_t ws_bytes, void *stream);

/* ---- compute_split_plan / partial_pary_search (split.py) ---------------- */

/* _fill_plan_kernel (split.py:52-88) for boundaries 0..s (arrays of s+1).
 * method 0: one binary search per boundary; method 1: the paper's batched
 * search — a CTA contracts the shared h-range of a run of consecutive
 * boundaries, stages the prefix windows in shared memory and finishes each
 * boundary there.  Both are bit-identical to the reference on the same
 * prefix arrays.  h_w has the weight dtype.  Replaces split.py:102. */
int ak_split_plan(const double *lprefix, uint64_t nl, const double *hprefix, uint64_t nh,
                  const void *h_w, int dtype, uint64_t n_total, uint64_t s, double avg,
                  int64_t *lcounts, int64_t *hcounts, double *spills, int method, void *stream);

/* [sync] partial_pary_search (split.py:190-213): lower-bound index of each
 * sorted query in the sorted haystack; validates sortedness
 * (AK_ERR_UNSORTED_INPUT) and p >= 3 (AK_ERR_VALUE).  Replaces split.py:209. */
int ak_partial_pary_search(const double *hay, uint64_t n, const double *q, uint64_t m,
                           uint32_t p, int64_t *out, void *stream);

/* ---- pack (pack.py) ----------------------------------------------------- */

/* _pack_range / _chunked_pack_range (pack.py:30-159) for sections
 * sec_first..sec_last (1-based, inclusive): the reference's per-section
 * sweep, bit-identical to it on the same partition and plan.  Lists as
 * written by ak_partition (int64 1-based indices, weights in `dtype`);
 * `rows` is a table in the layout of `dtype`; out_spills (may be NULL) gets
 * each section's outgoing residual.  chunk_capacity 0 = plain sweep, else the
 * staged variant (one warp per section stages l/h chunks coalesced into
 * shared memory).  Replaces pack.py:184/192. */
int ak_pack_sections(const int64_t *l_idx, const void *l_w, uint64_t nl, const int64_t *h_idx,
                     const void *h_w, uint64_t nh, int dtype, const int64_t *lcounts,
                     const int64_t *hcounts, const double *spills, uint64_t s,
                     uint64_t sec_first, uint64_t sec_last, double avg, void *rows,
                     double *out_spills, uint32_t chunk_capacity, void *stream);

/* ---- fused construction (psa_construct / vose_construct) ---------------- */

size_t ak_build_workspace_bytes(uint64_t n, int dtype);
/* psa_construct (pack.py:255-277) as one fused device pipeline over the
 * weights: classify + tile scan with decoupled look-back, coarse merge of
 * the tile prefix boundaries, and a tile-owner pack that resolves every
 * light's alias and every heavy's threshold from the prefix sums (see
 * DESIGN.md).  Alias indices equal the sequential Vose order; thresholds are
 * double-double accurate.  `total` is WeightSet.total.  `rows` gets the
 * table in the layout of `dtype`.  Asynchronous; stats (nl, nh, tiles) are
 * readable afterwards with ak_build_stats. */
/* Limit: n < 2^32 - 1 for both dtypes (u32 aliases in f32 rows, u32 item ids
 * in the pack's merge windows); larger n returns AK_ERR_VALUE. */
int ak_build_psa(const void *w, int dtype, uint64_t n, double total, void *rows, void *ws,
                 size_t ws_bytes, void *stream);
/* ak_build_psa with the bucket size avg given instead of total/n (the PSA+
 * residual is built with the global average, pack.py:297-299). */
int ak_build_psa_avg(const void *w, int dtype, uint64_t n, double avg, void *rows, void *ws,
                     size_t ws_bytes, void *stream);
/* [sync] Light/heavy counts and tile count of the last ak_build_psa on ws. */
int ak_build_stats(const void *ws, uint64_t n, uint64_t *nl, uint64_t *nh, uint64_t *tiles,
                   void *stream);

/* ---- PSA+ (greedy_prepack, partition.py:134-282; pack.py:280-305) ------- */

size_t ak_prepack_workspace_bytes(uint64_t n, uint32_t block_size);
/* [sync] _greedy_kernel (partition.py:134-227): per block of block_size items,
 * exactly-full items fill their own rows; if the block holds >= threshold
 * lights (w < avg) and heavies (w > avg) they are paired by the block-local
 * sequential order until one side runs out.  `rows` (table layout of dtype,
 * zeroed here) gets every handled row; the leftovers, in item order, go to
 * res_idx (1-based) / res_w (f64; the partially consumed heavy carries its
 * residual); *nres_out / *nwritten_out their counts.  Replaces the
 * _greedy_kernel_nb call (partition.py:253). */
int ak_greedy_prepack(const void *w, int dtype, uint64_t n, double avg, uint32_t block_size,
                      uint32_t threshold, void *rows, int64_t *res_idx, double *res_w,
                      uint64_t *nres_out, uint64_t *nwritten_out, void *ws, size_t ws_bytes,
                      void *stream);
/* The residual's table (f64 rows over residual positions 1..nres, built with
 * ak_build_psa_avg on res_w) written into the final table at res_idx, aliases
 * mapped back to item ids (pack.py:297-299). */
int ak_residual_scatter(const void *res_rows, const int64_t *res_idx, uint64_t nres, double avg,
                        int dtype, void *rows, void *stream);
/* ak_greedy_prepack with the row clearing optional (clear_rows = 0: rows the
 * prepack does not pair keep their contents; psa_plus fills them all). */
int ak_greedy_prepack_ex(const void *w, int dtype, uint64_t n, double avg, uint32_t block_size,
                         uint32_t threshold, int clear_rows, void *rows, int64_t *res_idx,
                         double *res_w, uint64_t *nres_out, uint64_t *nwritten_out, void *ws,
                         size_t ws_bytes, void *stream);
/* ak_residual_scatter that also returns how many rows it wrote with a
 * nonzero alias (a written bucket): with the prepack's own count, PSA+'s
 * "every bucket written" check (pack.py:303-304) without a pass over the
 * table. */
int ak_residual_scatter_count(const void *res_rows, const int64_t *res_idx, uint64_t nres,
                              double avg, int dtype, void *rows, uint64_t *written, void *stream);
/* PSA+'s residual construction (pack.py:296-305: the forwarded items go
 * through PSA with the global average) fused with the scatter: the k residual
 * weights res_w (f64, 16-byte aligned, in item order) are built as by
 * ak_build_psa_avg, and each residual row r is written straight into the
 * final table `rows` (out_dtype AK_F32 / AK_F64) at res_idx[r] - 1 with alias
 * res_idx[alias - 1], thresholds rounded as ak_residual_scatter rounds them.
 * *written = the rows written (k when every residual bucket is filled).
 * Equals ak_build_psa_avg + ak_residual_scatter_count without the
 * intermediate residual table.  ws: ak_build_workspace_bytes(k, AK_F64). */
int ak_build_psa_residual(const double *res_w, uint64_t k, double avg, const int64_t *res_idx,
                          int out_dtype, void *rows, uint64_t *written, void *ws, size_t ws_bytes,
                          void *stream);

/* ---- sampling (sample.py) ----------------------------------------------- */

/* _fill_samples (sample.py:73-84) over m draws with counters ctr0..: draw i
 * uses uniform(ctr0+i, stream_id, seed) (AK_RNG_REFERENCE, bit-exact) and
 * the bucket rule on rows [lo, lo+span); out int64 1-based.  Replaces
 * sample.py:110. */
int ak_sample_naive(const void *rows, int dtype, uint64_t n, double avg, uint64_t lo,
                    uint64_t span, uint64_t seed, uint64_t stream_id, uint64_t ctr0, uint64_t m,
                    int64_t *out, int rng_mode, void *stream);
/* ak_sample_naive with the output index dtype chosen (AK_I64 / AK_I32). */
int ak_sample_naive_out(const void *rows, int dtype, uint64_t n, double avg, uint64_t lo,
                        uint64_t span, uint64_t seed, uint64_t stream_id, uint64_t ctr0, uint64_t m,
                        void *out, int out_dtype, int rng_mode, void *stream);
/* The bucket rule fed explicit f64 uniforms (tests/test_sample.py:20-25):
 * the "identical uniform variates -> identical indices" parity hook. */
int ak_sample_from_uniforms(const void *rows, int dtype, uint64_t n, double avg, uint64_t lo,
                            uint64_t span, const double *u, uint64_t m, int64_t *out,
                            void *stream);
/* number of sections after clamping S to n_rows (sample.py:213-214) */
uint64_t ak_num_sections(uint64_t n_rows, uint64_t S);
/* [host] assign_subtree (sample.py:222-240) / assign_sections (203-219):
 * communication-free binomial section counts, bit-exact with the reference
 * (host libm log/sqrt/pow, round-half-even).  counts_out sized b-a. */
int ak_assign_subtree(uint64_t n_rows, uint64_t S, uint64_t seed, uint64_t stream_id,
                      uint64_t a, uint64_t b, uint64_t m, int64_t *counts_out);
/* sectioned_sample (sample.py:243-267) for sections [first, first+count):
 * section j draws counts[j] samples on derive_stream(seed, stream_id, j,
 * SALT_SECTION) with counters ctr0.., confined to its rows, which a CTA
 * stages in shared memory with a bulk async copy; out[offsets[j] - out_base
 * + i].  counts/offsets are device int64 arrays indexed by absolute section. */
int ak_sample_sectioned(const void *rows, int dtype, uint64_t n, double avg, uint64_t S,
                        const int64_t *counts, const int64_t *offsets, uint64_t first,
                        uint64_t count, uint64_t seed, uint64_t stream_id, uint64_t ctr0,
                        int64_t *out, int64_t out_base, int rng_mode, void *stream);
/* ak_sample_sectioned with the output index dtype chosen (AK_I64 / AK_I32). */
int ak_sample_sectioned_out(const void *rows, int dtype, uint64_t n, double avg, uint64_t S,
                            const int64_t *counts, const int64_t *offsets, uint64_t first,
                            uint64_t count, uint64_t seed, uint64_t stream_id, uint64_t ctr0,
                            void *out, int out_dtype, int64_t out_base, int rng_mode, void *stream);

/* ---- verification / conversion ------------------------------------------ */

size_t ak_validate_workspace_bytes(uint64_t n);
/* [sync] validate_table (model.py:111-144): row invariants (finite,
 * 0 <= tw <= avg*(1+row_tol), alias in 1..n; the reference uses
 * row_tol = 1e-9) and per-item reconstructed mass (compensated f64 atomics)
 * -> rows_ok, worst relative error and its 1-based item. */
int ak_validate_table(const void *rows, int dtype, uint64_t n, const void *w, int w_dtype,
                      double avg, double row_tol, int *rows_ok, double *worst_rel,
                      int64_t *worst_item, void *ws, size_t ws_bytes, void *stream);
/* [sync] validate_table for the items [item_lo, item_hi): every row is
 * read (its donation may land in the range), the row invariants are checked
 * for the rows of the range, the per-item mass for the items of the range.
 * Ranks of a sharded validation take disjoint ranges and reduce the three
 * results (min ok, max worst, min worst item among the maxima); the union
 * equals ak_validate_table.  Workspace: ak_validate_workspace_bytes(range). */
int ak_validate_table_range(const void *rows, int dtype, uint64_t n, uint64_t item_lo,
                            uint64_t item_hi, const void *w, int w_dtype, double avg,
                            double row_tol, int *rows_ok, double *worst_rel, int64_t *worst_item,
                            void *ws, size_t ws_bytes, void *stream);
/* chi_square_test's sums (stats.py:84-121) over bins [0, m) of a counts
 * shard with their weights: out4 = {sum over kept bins of (c-e)^2/e, kept
 * bins, pooled observed, pooled expected}, e_i = draws * w_i / total_w, a
 * bin kept iff e_i >= 5 (device doubles; shards add up). */
int ak_chi2_partial(const int64_t *counts, const void *w, int w_dtype, uint64_t m,
                    double total_w, double draws, double *out4, void *stream);
/* [sync] frequency_counts (stats.py:25-32): counts[i] = #samples == i+1. */
int ak_frequency_counts(const int64_t *samples, uint64_t m, uint64_t n, int64_t *counts,
                        void *stream);
/* table rows <-> reference SoA (tw f64, alias int64) */
int ak_rows_to_soa(const void *rows, int dtype, uint64_t n, double *tw, int64_t *alias,
                   void *stream);
int ak_soa_to_rows(const double *tw, const int64_t *alias, uint64_t n, int dtype, void *rows,
                   void *stream);
/* Rows [first, first+count) as ALT1 file rows (io.py:21): 16 bytes each, f64
 * threshold then u64 alias, into out (device) — the streamed save_table's
 * widening of f32 tables, chunk by chunk. */
int ak_rows_to_alt1(const void *rows, int dtype, uint64_t n, uint64_t first, uint64_t count,
                    void *out, void *stream);
/* [sync] count of rows with alias == 0 (pack.py:275-276 check) */
int ak_count_unwritten(const void *rows, int dtype, uint64_t n, uint64_t *unwritten,
                       void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ALIASKIT_B200_H */
