/* simjoin_b200.h -- C ABI of libsjb200.so, the B200 (sm_100a) implementation
 * of the reference's cosine-threshold tensor join hot path.
 *
 * Conventions (kept from the reference's _kernelcore.h:6-25):
 *   - raw pointers + 64-bit sizes, row-major contiguous fp32 rows, uint64_t
 *     offsets; outputs are caller-allocated with an explicit capacity and the
 *     exact count is reported so the caller can retry (the reference's
 *     count + capacity + resume protocol, _ckern.pyx:165-175, 194-211).
 *   - Pointers named d_* are DEVICE pointers; `stream` is a cudaStream_t
 *     (passed as void* so this header needs no CUDA include).
 *   - Every entry point returns an int status: SJB_OK (0) or a negative
 *     SJB_E_* code; sjb_last_error() returns a message for the calling
 *     thread.  Calls are re-entrant and safe on distinct devices/streams.
 *   - No torch types cross this boundary.
 *
 * Reference paths are relative to /root/reference/pkg/src/simjoin/.
 */
#ifndef SIMJOIN_B200_H
#define SIMJOIN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SJB_OK 0
#define SJB_E_INVALID (-1)     /* bad argument (shape, dim, capacity) */
#define SJB_E_CUDA (-2)        /* CUDA runtime error */
#define SJB_E_UNSUPPORTED (-3) /* shape this build does not handle */

#define SJB_TILE_ROWS 256

/* ---- library ---------------------------------------------------------- */
int sjb_version(void);
const char* sjb_last_error(void);
/* SM count of `device` (for sizing grids/workspaces). */
int sjb_sm_count(int device);

/* Number of kernels this library has launched in this process (all
 * threads); lets callers count the GPU launches inside a timed region. */
int64_t sjb_launch_count(void);

/* Padded reduction depth of the 16-bit operand image for `dim`: a multiple of
 * 16 for dim <= 128, of 64 above (K-streaming kernel). */
int64_t sjb_kpad(int64_t dim);
/* Elements of the 16-bit operand image (bf16 for kpad <= 128, fp16 above) of an n-row relation: n rounded up to a
 * multiple of 512 rows, times kpad.  Layout: 256-row tiles, each
 * [k-group (kpad/8)][row (256)][8 elements] (UMMA K-major, no swizzle). */
int64_t sjb_operand_elems(int64_t n, int64_t dim);
/* 256-row tiles of that image (= entries of a d_tile_err array). */
int64_t sjb_tile_count(int64_t n);

/* fp16 rounding-error outputs of the prep functions below (both optional,
 * written only together with d_out16):
 *   d_row_err[i]  (n floats)  >= ||fp16(x_i) - x_i||_2 of canonical row x_i
 *   d_tile_err[t] (sjb_tile_count(n) floats) = max of d_row_err over tile t
 * They let the join use a per-row filter band (sjb_join_args.left_row_err /
 * right_tile_err) instead of the worst-case sjb_default_band. */

/* ---- prefetch stage: embedding + normalise-and-cast -------------------- */

/* Row L2 normalisation, bitwise equal to sj_normalize_rows
 * (_kernelcore.h:8, _kernelcore.c:52-87): fp64 sequential sum of squares,
 * zero rows repaired (component 0 := 1), fp64 divide, fp32 store.
 * d_in may equal d_out32 (in place).  d_out16 (optional, may be NULL) gets the
 * 16-bit operand image (sjb_operand_elems elements; bf16 for kpad <= 128, fp16
 * above).  *d_repaired (optional
 * device u64) is incremented by the number of repaired rows. */
int sjb_normalize_rows(const float* d_in, int64_t n, int64_t dim, float* d_out32,
                       void* d_out16, unsigned long long* d_repaired, float* d_row_err,
                       float* d_tile_err, void* stream);

/* Lookup-model prefetch fused with the normalisation: relation row i is
 * table row d_index[i] (LookupModel._vector, embedding.py:143-152, then
 * normalize_rows); outputs as sjb_normalize_rows. */
int sjb_gather_normalize_rows(const float* d_table, const int64_t* d_index, int64_t n,
                              int64_t dim, float* d_out32, void* d_out16,
                              unsigned long long* d_repaired, float* d_row_err,
                              float* d_tile_err, void* stream);

/* Operand image of rows used AS GIVEN (no normalisation): the 16-bit tiled
 * image (sjb_operand_elems elements) of n x dim fp32 rows.  For callers that
 * hand over rows they already normalised (the kernel-backend nlj_rows
 * contract, _ckern.pyx:179-212; EmbeddedRelation.normalized) -- the filter
 * band must then cover those rows' norms (sjb_default_band scaled by the
 * largest norms; see kernels.nlj_rows). */
int sjb_cast_rows(const float* d_in, int64_t n, int64_t dim, void* d_out16, void* stream);

/* bf16 relation prep for the raw-operand wide filter (dim > 128): d_in is
 * n x dim bf16 (row-major).  d_out32 = canonical normalised fp32 rows
 * (bitwise sj_normalize_rows of the rows' exact fp32 values); d_out16 = the
 * RAW bf16 rows in the tiled operand layout (sjb_operand_elems elements; a
 * repaired row has component 0 = 1 like the reference's); d_inv_norm
 * (sjb_operand_elems / kpad floats: rows padded to 512, 0 past n) =
 * RN(1 / ||x_i||). */
int sjb_prepare_bf16(const void* d_in, int64_t n, int64_t dim, float* d_out32, void* d_out16,
                     float* d_inv_norm, unsigned long long* d_repaired, void* stream);

/* Filter band of the raw-operand mode: the bf16 products are exact, so
 * |approx - canonical| is fp32 accumulation (both sums) plus the inverse
 * norms' and the epilogue products' roundings: 4 dim 2^-24 + 8 2^-24 + 2e-6. */
float sjb_raw_band(int64_t dim);

/* 1 when the library was built with the measured-and-rejected A/B kernels
 * (-DSJB_AB_KERNELS=1: SJB_FILTER=pair|ts, SJB_RBLOCK=512,
 * SJB_WIDE_RECHECK=fused|tile); 0 in the default build, where those
 * switches fail with SJB_E_UNSUPPORTED. */
int sjb_ab_kernels(void);

/* Diagnostics of the dense (deferred) recheck: copies and zeroes 16 counters
 * -- dense / big-row / union-overflow / low-density blocks, candidates in
 * dense and in sparse blocks, summed dense union sizes, then SM cycles per
 * block phase.  Only in a build with -DSJB_BLK_STATS=1; otherwise
 * SJB_E_UNSUPPORTED. */
int sjb_debug_blk_stats(int64_t* out16);

/* Row norms (sj_row_norms, _kernelcore.h:9). */
int sjb_row_norms(const float* d_m, int64_t n, int64_t dim, float* d_out, void* stream);

/* FNV-1a-64 of packed tokens XOR xor_seed (sj_fnv1a64, _kernelcore.h:6;
 * SyntheticModel._stream_seed, embedding.py:87-88).  Token t is
 * d_bytes[d_offs[t], d_offs[t+1]). */
int sjb_fnv1a64_many(const uint8_t* d_bytes, const int64_t* d_offs, int64_t n,
                     uint64_t xor_seed, uint64_t* d_out, void* stream);

/* Synthetic model rows from stream seeds (sj_synthetic_fill, _kernelcore.h:7;
 * SyntheticModel._embed_into, embedding.py:95-107), normalised per the model.
 * d_out16 optional as above. */
int sjb_synthetic_fill_many(const uint64_t* d_seeds, int64_t n, int64_t dim, float* d_out32,
                            void* d_out16, float* d_row_err, float* d_tile_err, void* stream);

/* FastText-style subword model (cfg3; no reference counterpart, see
 * DESIGN.md): row = mean of table rows of the word hash and every
 * minn..maxn-gram of '<'w'>' (fnv1a64 mod n_buckets).  normalize != 0 also
 * applies sjb_normalize_rows and writes the 16-bit operand image (d_out16 optional). */
int sjb_subword_embed(const uint8_t* d_bytes, const int64_t* d_offs, int64_t n,
                      const float* d_table, int64_t n_buckets, int64_t dim, int minn,
                      int maxn, int normalize, float* d_out32, void* d_out16,
                      unsigned long long* d_repaired, float* d_row_err, float* d_tile_err,
                      void* stream);

/* ---- the fused join --------------------------------------------------- */

typedef struct sjb_join_args {
  int64_t n_left, n_right, dim;
  float theta;          /* inclusive: a pair matches iff canonical sim >= theta */
  float band;           /* fp16 filter margin; candidates have approx >= theta - band */
  int64_t cand_cap;     /* candidate buffer entries (workspace) */
  int64_t out_cap;      /* capacity of lefts/rights/sims */
  uint64_t left_base;   /* added to emitted left offsets (R shards) */
  int32_t grid;         /* 0 = one CTA per SM */
  int32_t tiles_per_chunk; /* 0 = automatic */
  void* ev_filter_begin;   /* optional cudaEvent_t recorded around the filter */
  void* ev_filter_end;     /* kernel on `stream` (profiling hook), or NULL */
  /* Optional per-row band (both or neither): the left relation's d_row_err
   * and the right relation's d_tile_err from the prep functions.  Row i of
   * S tile t then keeps pairs with approx >= max(theta - band,
   * theta - b_it), b_it = slack + (1+1e-6)(e_i + E_t) + e_i E_t,
   * slack = sjb_accum_slack(dim): Cauchy-Schwarz on the measured fp16
   * rounding errors, so no true match is dropped. */
  const float* left_row_err;
  const float* right_tile_err;
  /* Canonical recheck placement (dim <= 128): 0 = fused into the filter (two
   * warps recheck while the S chunk is in L2; best for sparse results),
   * 1 = deferred to a full-occupancy kernel after the filter (best when
   * candidates are dense, e.g. > 2e-4 of the pairs).  Same result. */
  int32_t recheck;
  /* Raw-operand mode (bf16 relations, sjb_prepare_bf16; dim > 128): both
   * relations' RN(1/||x||) from the prep; the operand images then hold the
   * raw bf16 rows and the filter normalises after the GEMM.  Use
   * band = sjb_raw_band(dim).  NULL: normalised operands (default). */
  const float* left_inv_norm;
  const float* right_inv_norm;
  /* Similarity values (raw-operand mode only): 0 = canonical (every
   * candidate rechecked, bitwise sj_dot_seq; default), 1 = tensor: pairs
   * with approx >= theta + band are emitted with the epilogue similarity
   * (|approx - canonical| < band, measured ~1e-6), only pairs within the
   * band are rechecked canonically.  The pair SET is exact either way. */
  int32_t sims_mode;
  /* CTAs of this filter launch (dim <= 128 kernel; 0 = the plan's grid,
   * i.e. args->grid or one per SM).  Fewer CTAs than the plan leave SMs free
   * for kernels that must run beside the filter (NCCL's all-gathers of later
   * S rounds); the segments of the plan's other CTAs stay empty. */
  int32_t launch_grid;
} sjb_join_args;

typedef struct sjb_join_info {
  int64_t n_matches;    /* exact number of matches */
  int64_t n_candidates; /* exact number of filter candidates */
  int64_t cand_needed;  /* candidate capacity that avoids overflow on retry */
  int32_t overflow;     /* 1: candidates or outputs overflowed -> retry */
  int32_t grid;         /* CTAs the filter kernel ran with */
} sjb_join_info;

/* Workspace bytes needed by sjb_join_prepared for these args. */
int64_t sjb_join_workspace_bytes(const sjb_join_args* args);

/* Default (provably sufficient) band for `dim`: fp16 rounding of unit
 * vectors (2u+u^2, u = 2^-8) plus fp32 accumulation slack. */
float sjb_default_band(int64_t dim);
/* The accumulation part of that band (+ 1e-6 for the fp32 cutoff
 * arithmetic): the `slack` of the per-row band (sjb_join_args). */
float sjb_accum_slack(int64_t dim);

/* Join two prepared (normalised) relations on the device; asynchronous.
 * d_l32/d_r32: canonical fp32 rows; d_l16/d_r16: 16-bit operand images.
 * Replaces tensor_join's tile loop (join.py:338-359: tile_similarity +
 * threshold_scan + MatchSink.merge) with filter -> canonical recheck ->
 * row bucketing -> per-row sort.  Writes the canonical MatchSet columns to
 * d_lefts/d_rights/d_sims and the sjb_join_info fields to d_info (device
 * memory, 5 x 8 bytes) without synchronising. */
int sjb_join_prepared_async(const float* d_l32, const void* d_l16, const float* d_r32,
                            const void* d_r16, const sjb_join_args* args, void* d_workspace,
                            int64_t workspace_bytes, uint64_t* d_lefts, uint64_t* d_rights,
                            float* d_sims, void* d_info, void* stream);

/* Synchronous form: as above, then waits on `stream` and copies the info to
 * the host struct *info. */
/* The same join in steps, so the filter can start on the first S tiles while
 * later ones are still being copied or broadcast (one stream; args and
 * workspace identical across the steps of one join):
 *   sjb_join_begin        zero the counters (and empty the candidate slots)
 *   sjb_join_filter_tiles filter + canonical recheck of S tiles
 *                         [tile_begin, tile_end) (256-row tiles; ranges of
 *                         one join must be disjoint and together cover S;
 *                         only those S rows must be prepared when it runs)
 *   sjb_join_finish       (deferred canonical recheck,) bucket, sort and emit
 *                         the MatchSet; writes d_info
 * sjb_join_prepared_async = begin + filter_tiles(all) + finish. */
int sjb_join_begin(const sjb_join_args* args, void* d_workspace, int64_t workspace_bytes,
                   void* stream);
int sjb_join_filter_tiles(const float* d_l32, const void* d_l16, const float* d_r32,
                          const void* d_r16, const sjb_join_args* args, void* d_workspace,
                          int64_t workspace_bytes, int64_t tile_begin, int64_t tile_end,
                          void* stream);
int sjb_join_finish(const float* d_l32, const float* d_r32, const sjb_join_args* args,
                    void* d_workspace, int64_t workspace_bytes, uint64_t* d_lefts,
                    uint64_t* d_rights, float* d_sims, void* d_info, void* stream);

int sjb_join_prepared(const float* d_l32, const void* d_l16, const float* d_r32,
                      const void* d_r16, const sjb_join_args* args, void* d_workspace,
                      int64_t workspace_bytes, uint64_t* d_lefts, uint64_t* d_rights,
                      float* d_sims, sjb_join_info* info, void* stream);

/* ---- dense kernels of the reference backend API ------------------------ */

/* out[i*ldo+j] = canonical dot(left row i, packed column j)
 * (sj_tile_dot, _kernelcore.h:13-14; bt = pack_transpose, dim x nr). */
int sjb_tile_dot(const float* d_left, int64_t lda, const float* d_bt, int64_t ldb, int64_t nl,
                 int64_t nr, int64_t dim, float* d_out, int64_t ldo, void* stream);

/* out[i] = canonical dot(a, row i) (sj_dots_vm, _kernelcore.h:11). */
int sjb_dots_vm(const float* d_a, const float* d_m, int64_t n, int64_t dim, float* d_out,
                void* stream);

/* out[i] = cosine of a and row i with the reference's arithmetic (cosine_vm,
 * linalg.py:70-84): sj_dots_vm / (fp32(sj_row_norms(a)) * sj_row_norms(row i)),
 * fp32 multiply then fp32 divide.  *d_flags (device int, zeroed by the
 * caller) gets bit 0 if ||a|| == 0 and bit 1 if some row norm is 0 -- the
 * reference raises ZeroVector in both cases.  Used by e_selection
 * (join.py:145-179) and top_k (embedding.py:218-231). */
int sjb_cosine_vm(const float* d_a, const float* d_m, int64_t n, int64_t dim, float* d_out,
                  int* d_flags, void* stream);

/* Row-major threshold scan of a dense nl x nr buffer (sj_scan_count +
 * sj_scan_fill, _kernelcore.h:15-18).  Pass 1 (outputs NULL): *count = hits.
 * Pass 2: fills up to cap hits in row-major order.  Synchronous. */
int sjb_scan_hits(const float* d_buf, int64_t nl, int64_t nr, float theta, uint64_t left0,
                  uint64_t right0, uint64_t* d_lefts, uint64_t* d_rights, float* d_sims,
                  int64_t cap, int64_t* count, void* d_workspace, int64_t workspace_bytes,
                  void* stream);
int64_t sjb_scan_hits_workspace_bytes(int64_t nl);

/* The matches file (cli._write_matches, cli.py:105-108; _fmt_sim 99-102):
 * line i = "<lefts[i]>,<rights[i]>,<sim>\n", <sim> the shortest positional
 * decimal that reads back as the same float32 (numpy
 * format_float_positional(unique=True, trim="-")); "-0", "inf", "nan" as
 * numpy prints them.  Replaces the per-line Python formatting loop.
 * Layout (synchronous): computes the line offsets into the workspace and
 * *out_bytes = file size.  Write (asynchronous): the file bytes into d_out,
 * using the workspace of a layout call on the same columns. */
int64_t sjb_matches_csv_workspace_bytes(int64_t n);
int sjb_matches_csv_layout(const uint64_t* d_lefts, const uint64_t* d_rights,
                           const float* d_sims, int64_t n, void* d_workspace,
                           int64_t workspace_bytes, int64_t* out_bytes, void* stream);
int sjb_matches_csv_write(const uint64_t* d_lefts, const uint64_t* d_rights,
                          const float* d_sims, int64_t n, const void* d_workspace,
                          int64_t workspace_bytes, uint8_t* d_out, int64_t out_cap,
                          void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SIMJOIN_B200_H */
