// sjb_capi.cu -- extern "C" boundary of libsjb200.so (declared in
// include/simjoin_b200.h) and the host-side orchestration of the join
// pipeline.  Built as ONE translation unit with the kernel sources.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "../../include/simjoin_b200.h"
#include "sjb_common.cuh"
#include "sjb_join.cu"
// The measured-and-rejected A/B kernels (DESIGN.md "Measured and rejected":
// TS-mode filter, CTA-pair filter, 512-row R blocks, the wide filter with
// fused recheck warps, the per-tile staged wide recheck) are built only with
// -DSJB_AB_KERNELS=1 (SJB_NVCC_EXTRA); the default library holds the
// measured-best kernels.
#ifndef SJB_AB_KERNELS
#define SJB_AB_KERNELS 0
#endif
#if SJB_AB_KERNELS
#include "sjb_join_ts.cu"
#include "sjb_join2.cu"
#endif
#include "sjb_join3.cu"
#include "sjb_join4.cu"
#include "sjb_post.cu"
#include "sjb_prep.cu"
#include "sjb_fmt.cu"

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define SJB_CK(expr)                                                                       \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(SJB_E_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),      \
                  __FILE__, __LINE__);                                                     \
  } while (0)

#define SJB_CK_LAUNCH(name)                                                                \
  do {                                                                                     \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                    \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess)                                                                 \
      return fail(SJB_E_CUDA, "launch of %s failed: %s", name, cudaGetErrorString(e_));    \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

int max_dyn_smem(int dev) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

// Sub-tile rows for the prep kernels: as many of the 128 tile rows as fit in
// ~100 KB of smem (so 2 CTAs fit per SM), multiple of 32.
int prep_sub_rows(int64_t dim) {
  const int64_t pitch = dim | 1;
  int sub = 128;
  while (sub > 32 && (int64_t)sub * pitch * 4 > 100 * 1024) sub >>= 1;
  return sub;
}

int set_smem_attr(const void* fn, int bytes) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess)
    return fail(SJB_E_CUDA, "cudaFuncSetAttribute(%d B) failed: %s", bytes, cudaGetErrorString(e));
  return SJB_OK;
}

// ---------------------------------------------------------------- plan
struct JoinPlan {
  int kpad, stages, a_bufs, a_tiles, grid, tiles_per_chunk, n_ablk, n_btiles;
  int64_t n_items;
  uint32_t smem;
  uint64_t seg_cap;
  bool pair;  // CTA-pair (cta_group::2) filter kernel
  bool ts;    // R block in tensor memory (sjb_join_ts.cu; opt-in A/B, SJB_FILTER=ts)
  bool wide;  // K-streaming kernel (kpad > 128)
  bool wide_fused;        // wide: recheck inside the filter (A/B only)
  bool defer;             // d <= 128: row-grouped recheck after the filter (dense joins)
  bool wide_rows;         // wide, raw operands, canonical sims: the CTA-pair filter emits candidates
                          // only; they are grouped by left row and rechecked by staged warps
  int64_t tile_stride;    // wide, separate recheck: tile offsets per CTA
};

// Recheck placement for d <= 128: args->recheck (0 fused, 1 deferred); the
// SJB_RECHECK environment variable ("fused" / "deferred") overrides it.
bool use_deferred_recheck(const sjb_join_args* a) {
  const char* f = getenv("SJB_RECHECK");
  if (f != nullptr && strcmp(f, "fused") == 0) return false;
  if (f != nullptr && strcmp(f, "deferred") == 0) return true;
  return a->recheck == 1;
}

// Deferred recheck through recheck_rows_kernel (sorted rows, bulk-copied S
// rows) where its 1-D copies apply: dim % 4 == 0, 16-byte aligned rows;
// SJB_DENSE_RECHECK=grouped keeps the per-lane gather kernel (A/B).
constexpr int kRowsSmemMax = 227 * 1024;
bool use_rows_recheck(const sjb_join_args* a, const float* l32, const float* r32) {
  const char* f = getenv("SJB_DENSE_RECHECK");
  if (f != nullptr && strcmp(f, "grouped") == 0) return false;
  return a->dim % 4 == 0 && a->dim <= 128 &&
         ((reinterpret_cast<uintptr_t>(l32) | reinterpret_cast<uintptr_t>(r32)) & 15) == 0 &&
         sjb::rows_warp_smem((int)a->dim, false) + 128 <= kRowsSmemMax;
}

// Dense recheck variant (A/B): 0 cluster-blocked rows (default), 1 one warp
// per sorted row (SJB_DENSE_RECHECK=rows); "grouped" = use_rows_recheck false.
int dense_mode() {
  const char* f = getenv("SJB_DENSE_RECHECK");
  return (f != nullptr && strcmp(f, "rows") == 0) ? 1 : 0;
}

bool use_wide_fused() {
  const char* f = getenv("SJB_WIDE_RECHECK");
  return f != nullptr && strcmp(f, "fused") == 0;
}

// K-streaming plan (kpad > 128): 256 x 256 output tiles, 64-element K chunks.
int make_wide_plan(const sjb_join_args* a, JoinPlan* pl, int sms, int max_smem) {
  namespace W = sjb::wide;
  pl->wide = true;
  pl->wide_fused = use_wide_fused();
  pl->a_bufs = 0;
  pl->a_tiles = 1;
  int stages = 0;
  const bool tol = a->sims_mode == 1;
  while (stages < W::kMaxStages && (int)W::smem_bytes(stages + 1, tol) <= max_smem) stages++;
  if (stages < 2) return fail(SJB_E_UNSUPPORTED, "not enough shared memory for the wide kernel");
  pl->stages = stages;
  pl->smem = W::smem_bytes(stages, tol);
  pl->n_ablk = (int)sjb::ceil_div(a->n_left, sjb::kTileRows);
  pl->n_btiles = (int)sjb::ceil_div(a->n_right, sjb::kTileRows);
  int tpc = a->tiles_per_chunk;
  if (tpc <= 0) {
    const int64_t work = (int64_t)pl->n_ablk * pl->n_btiles;
    int64_t t = work / (4LL * sms);
    tpc = (int)(t < 1 ? 1 : (t > 32 ? 32 : t));
  }
  pl->tiles_per_chunk = tpc;
  pl->n_items = (int64_t)pl->n_ablk * sjb::ceil_div(pl->n_btiles, tpc);
  int grid = a->grid > 0 ? a->grid : sms;
  if ((int64_t)grid > pl->n_items) grid = (int)(pl->n_items > 0 ? pl->n_items : 1);
  pl->grid = grid;
  pl->seg_cap = (uint64_t)(a->cand_cap / grid);
  pl->tile_stride = pl->wide_fused ? 0 : W::tile_stride(pl->n_ablk, pl->n_btiles, grid, tpc);
  return SJB_OK;
}

bool use_pair_filter() {
  const char* f = getenv("SJB_FILTER");
  return f != nullptr && strcmp(f, "pair") == 0;
}

int ab_missing(const char* what) {
  return fail(SJB_E_UNSUPPORTED, "%s is an A/B kernel: rebuild with SJB_NVCC_EXTRA=-DSJB_AB_KERNELS=1",
              what);
}

#if SJB_AB_KERNELS
// CTA-pair plan: pair R block = 512 rows, pair S tile = 128 rows.
int make_pair_plan(const sjb_join_args* a, JoinPlan* pl, int sms, int max_smem) {
  namespace P = sjb::pair;
  pl->pair = true;
  pl->a_bufs = 2;
  pl->a_tiles = 1;
  const sjb::pair::Layout L0 = P::layout(pl->kpad, 0);
  int stages = (int)((max_smem - (int)L0.total - 3 * 8 * 12) / (int)L0.b_bytes);
  if (stages > 12) stages = 12;
  if (stages < 3) return fail(SJB_E_UNSUPPORTED, "not enough shared memory for the pair kernel");
  pl->stages = stages;
  pl->smem = P::layout(pl->kpad, stages).total;
  pl->n_ablk = (int)sjb::ceil_div(a->n_left, 2 * P::kARows);
  pl->n_btiles = (int)sjb::ceil_div(a->n_right, P::kUmmaN);
  const int pairs_max = sms / 2;
  int tpc = a->tiles_per_chunk;
  if (tpc <= 0) {
    const int64_t work = (int64_t)pl->n_ablk * pl->n_btiles;
    int64_t t = work / (4LL * pairs_max);
    tpc = (int)(t < 1 ? 1 : (t > 256 ? 256 : t));
  }
  pl->tiles_per_chunk = tpc;
  pl->n_items = (int64_t)pl->n_ablk * sjb::ceil_div(pl->n_btiles, tpc);
  int pairs = a->grid > 0 ? a->grid / 2 : pairs_max;
  if (pairs < 1) pairs = 1;
  if ((int64_t)pairs > pl->n_items) pairs = (int)(pl->n_items > 0 ? pl->n_items : 1);
  pl->grid = 2 * pairs;
  pl->seg_cap = (uint64_t)(a->cand_cap / pl->grid);
  return SJB_OK;
}
#endif

int make_plan(const sjb_join_args* a, JoinPlan* pl) {
  const int dev = current_device();
  const int sms = sjb_sm_count(dev);
  pl->kpad = (int)sjb_kpad(a->dim);
  pl->pair = false;
  pl->ts = false;
  pl->wide = false;
  pl->wide_fused = false;
  pl->tile_stride = 0;
  pl->defer = false;
  pl->wide_rows = false;
  const bool raw = a->left_inv_norm != nullptr || a->right_inv_norm != nullptr;
  if (raw && (a->left_inv_norm == nullptr || a->right_inv_norm == nullptr))
    return fail(SJB_E_INVALID, "raw-operand mode needs both relations' inverse norms");
  if (raw && pl->kpad <= 128)
    return fail(SJB_E_UNSUPPORTED, "raw-operand mode is for dim > 128 (the wide filter)");
  if (a->sims_mode == 1 && !raw)
    return fail(SJB_E_INVALID, "sims_mode 1 (tensor similarities) needs raw-operand mode");
  if (pl->kpad > 128) {
    if (int rc = make_wide_plan(a, pl, sms, max_dyn_smem(dev))) return rc;
    if (a->sims_mode == 1) pl->wide_fused = false;   // pending lists need the separate recheck
    if (!SJB_AB_KERNELS && pl->wide_fused) return ab_missing("SJB_WIDE_RECHECK=fused");
    {
      // A/B (SJB_WIDE_EXACT=rows), canonical sims on raw operands: the CTA-pair filter emits
      // candidates only and records each work item's segment offset; work items are then
      // rechecked in the filter's S-chunk-major order by warps that counting-sort 2048
      // candidates by left row and stage each distinct left row once beside 32 private S
      // rows (recheck_segments_sorted_kernel).  Bitwise the same result; measured slower at
      // the cfg4 slice (53 vs 48 ms): the filter falls 19.5 -> 15.2 ms, but the staged
      // recheck takes 34 ms vs 25.6 ms for the tile-group recheck -- it is bound by the
      // cp.async issue rate (one 512-byte LDGSTS per 8 cycles per SM, ~64 B/cycle), whatever
      // the candidate order (row-grouped: 27.5 ms; filter order by position: 29.8 ms) or
      // ring depth.  Default: the 1-CTA filter + tile-group recheck.
      const char* we = getenv("SJB_WIDE_EXACT");
      pl->wide_rows = raw && a->sims_mode == 0 && !pl->wide_fused && (pl->grid % 2) == 0 &&
                      (a->dim % 4) == 0 && a->out_cap >= a->cand_cap &&
                      we != nullptr && strcmp(we, "rows") == 0;
    }
    return SJB_OK;
  }
#if SJB_AB_KERNELS
  if (use_pair_filter()) return make_pair_plan(a, pl, sms, max_dyn_smem(dev));
#else
  if (use_pair_filter()) return ab_missing("SJB_FILTER=pair");
#endif
  // the row-grouped recheck stages candidates in the output-sized key buffer
  pl->defer = use_deferred_recheck(a) && a->out_cap >= a->cand_cap;
  const char* fe = getenv("SJB_FILTER");
  if (!SJB_AB_KERNELS && fe != nullptr && strcmp(fe, "ts") == 0) return ab_missing("SJB_FILTER=ts");
#if SJB_AB_KERNELS
  if (fe != nullptr && strcmp(fe, "ts") == 0) {
    // R block in tensor memory (A/B): one shared-memory image + B stages.
    // cfg2 filter 16.8 ms vs 16.45 for the SS kernel (MMA-only 14.65 in
    // both: the tensor pipe is power-bound, not shared-memory-bound)
    namespace T = sjb::ts;
    const int max_smem = max_dyn_smem(dev);
    const T::SmemLayout L0 = T::smem_layout(pl->kpad, 0);
    int stages = (int)((max_smem - (int)L0.total - 2 * 8 * 6) / (int)L0.tile_bytes);
    if (stages > 6) stages = 6;
    if (stages < 2) return fail(SJB_E_UNSUPPORTED, "not enough shared memory for 2 stages");
    pl->ts = true;
    pl->stages = stages;
    pl->a_bufs = 1;
    pl->a_tiles = 1;
    pl->smem = T::smem_layout(pl->kpad, stages).total;
    pl->n_ablk = (int)sjb::ceil_div(a->n_left, sjb::kTileRows);
  } else
#endif
  {
  // Shared memory: the resident R block is one 256-row tile (two M=128
  // halves per S tile).  SJB_RBLOCK=512 selects two-tile blocks (four halves
  // per S tile: half the S traffic per MMA; cfg2 filter 14.55 vs 15.2 ms
  // with emission disabled, 16.5 ms in full either way -- kept for A/B).
  // Within a block size, prefer a double-buffered block when that still
  // leaves 3 B stages; otherwise one buffer (reloaded between items).
  const int max_smem = max_dyn_smem(dev);
  const char* rbe = getenv("SJB_RBLOCK");
  int a_tiles = (rbe != nullptr && atoi(rbe) == 512) ? 2 : 1;
  if (!SJB_AB_KERNELS && a_tiles == 2) return ab_missing("SJB_RBLOCK=512");
  int stages = 0, a_bufs = 2;
  for (;; a_tiles--) {
    for (a_bufs = 2; a_bufs >= 1; a_bufs--) {
      sjb::JoinSmemLayout L0 = sjb::join_smem_layout(pl->kpad, 0, a_bufs, a_tiles);
      stages = (int)((max_smem - (int)L0.total) / (int)L0.tile_bytes);
      if (stages >= 3) break;
    }
    if (a_bufs < 1) a_bufs = 1;
    if (stages >= 2 || a_tiles == 1) break;
  }
  if (stages > 6) stages = 6;
  if (stages < 2) return fail(SJB_E_UNSUPPORTED, "not enough shared memory for 2 stages");
  pl->stages = stages;
  pl->a_bufs = a_bufs;
  pl->a_tiles = a_tiles;
  pl->smem = sjb::join_smem_layout(pl->kpad, stages, a_bufs, a_tiles).total;
  pl->n_ablk = (int)sjb::ceil_div(a->n_left, (int64_t)sjb::kTileRows * a_tiles);
  }
  pl->n_btiles = (int)sjb::ceil_div(a->n_right, sjb::kBN);
  int tpc = a->tiles_per_chunk;
  if (tpc <= 0) {
    const int64_t pairs = (int64_t)pl->n_ablk * pl->n_btiles;
    int64_t t = pairs / (4LL * sms);
    tpc = (int)(t < 1 ? 1 : (t > 64 ? 64 : t));
  }
  pl->tiles_per_chunk = tpc;
  pl->n_items = (int64_t)pl->n_ablk * sjb::ceil_div(pl->n_btiles, tpc);
  int grid = a->grid > 0 ? a->grid : sms;
  if ((int64_t)grid > pl->n_items) grid = (int)(pl->n_items > 0 ? pl->n_items : 1);
  pl->grid = grid;
  pl->seg_cap = (uint64_t)(a->cand_cap / grid);
  return SJB_OK;
}

// ------------------------------------------------------------ workspace
struct JoinWs {
  size_t cand, sims, cta, rowcount, rowoff, cursor, keys, bsums, bigrows, nbig, tiles, ncand,
      work, sig, desc, ccnt, total;
  size_t pend, pendn;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }


JoinWs join_ws_layout(const sjb_join_args* a, int grid, int64_t tile_stride) {
  JoinWs w;
  size_t o = 0;
  const size_t ccap = (size_t)(a->cand_cap > 0 ? a->cand_cap : 0);
  const size_t nl = (size_t)(a->n_left > 0 ? a->n_left : 0);
  const size_t ocap = (size_t)(a->out_cap > 0 ? a->out_cap : 0);
  const size_t nblocks = sjb::ceil_div((int64_t)nl, sjb::kScanBlock) + 1;
  w.cand = o;     o = align256(o + ccap * 8);
  w.sims = o;     o = align256(o + ccap * 4);
  w.cta = o;      o = align256(o + (size_t)grid * 8);
  w.rowcount = o; o = align256(o + nl * 4);
  w.rowoff = o;   o = align256(o + (nl + 1) * 8);
  w.cursor = o;   o = align256(o + (nl + 1) * 8);
  w.keys = o;     o = align256(o + ocap * 8);
  w.bsums = o;    o = align256(o + (nblocks + 1) * 8);
  w.bigrows = o;  o = align256(o + nl * 4);
  w.nbig = o;     o = align256(o + 16);
  w.tiles = o;    o = align256(o + (size_t)grid * (size_t)tile_stride * 4);
  w.ncand = o;    o = align256(o + 16);
  w.work = o;     o = align256(o + 16);
  w.sig = o;      o = align256(o + nl * 4);   // dense recheck: row signatures
  w.desc = o;     o = align256(o + nl * 8);   // dense recheck: block descriptors
  w.ccnt = o;     o = align256(o + nl * 4);   // dense recheck: candidates per row
  // tolerance emission: per-CTA pending slot lists + counts
  const bool tol = a->sims_mode == 1;
  w.pend = o;     o = align256(o + (tol ? ccap * 4 : 0));
  w.pendn = o;    o = align256(o + (tol ? (size_t)grid * 4 : 0));
  w.total = o;
  return w;
}

int grid_for(uint64_t n, int threads, int per_sm_blocks) {
  const int sms = sjb_sm_count(current_device());
  uint64_t g = (n + threads - 1) / threads;
  const uint64_t cap = (uint64_t)sms * per_sm_blocks;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// exclusive scan of n u32 counts into out[0..n] (u64) (+ optional copy)
int run_scan(const uint32_t* counts, int64_t n, uint64_t* out, uint64_t* out_copy,
             uint64_t* bsums, cudaStream_t st) {
  const int64_t nb = sjb::ceil_div(n, sjb::kScanBlock);
  if (nb > (int64_t)sjb::kScanBlock)
    return fail(SJB_E_UNSUPPORTED, "row scan supports at most %d rows",
                sjb::kScanBlock * sjb::kScanBlock);
  if (nb == 0) {
    SJB_CK(cudaMemsetAsync(out, 0, 8, st));
    if (out_copy) SJB_CK(cudaMemsetAsync(out_copy, 0, 8, st));
    return SJB_OK;
  }
  uint64_t* grand = bsums + nb;
  sjb::scan_reduce_kernel<<<(unsigned)nb, sjb::kScanThreads, 0, st>>>(counts, n, bsums);
  SJB_CK_LAUNCH("scan_reduce");
  sjb::scan_blocks_kernel<<<1, sjb::kScanThreads, 0, st>>>(bsums, nb, grand);
  SJB_CK_LAUNCH("scan_blocks");
  sjb::scan_down_kernel<<<(unsigned)nb, sjb::kScanThreads, 0, st>>>(counts, n, bsums, grand, out,
                                                                     out_copy);
  SJB_CK_LAUNCH("scan_down");
  return SJB_OK;
}

template <int KS, int AT>
int launch_filter_kat(const sjb::JoinParams& jp, int grid, uint32_t smem, cudaStream_t st) {
  if (int rc = set_smem_attr((const void*)sjb::join_filter_kernel<KS, AT>, (int)smem)) return rc;
  sjb::join_filter_kernel<KS, AT><<<grid, sjb::kJoinThreads, smem, st>>>(jp);
  SJB_CK_LAUNCH("join_filter");
  return SJB_OK;
}
template <int KS>
int launch_filter_ks(const sjb::JoinParams& jp, int grid, uint32_t smem, cudaStream_t st) {
#if SJB_AB_KERNELS
  if (jp.ts) {
    if (int rc = set_smem_attr((const void*)sjb::ts::filter_kernel<KS>, (int)smem)) return rc;
    sjb::ts::filter_kernel<KS><<<grid, sjb::ts::kThreads, smem, st>>>(jp);
    SJB_CK_LAUNCH("join_filter_ts");
    return SJB_OK;
  }
  if (jp.a_tiles == 2) return launch_filter_kat<KS, 2>(jp, grid, smem, st);
#endif
  return launch_filter_kat<KS, 1>(jp, grid, smem, st);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// The 16-bit operand image (sjb_operand_elems elements, 256-row tiles of
// [k-group][row][8]) as a 3-D tensor (256 elements = 32 rows x 8, 8 row
// blocks, kgroups * tiles); box {256, box_rows/32, box_kgroups (0: all)} =
// one [k-group][box_rows][8] block.  The 512 B inner extent keeps every
// request at full 32 B sectors (a 16 B inner box over-fetched 2x and issued
// ~900 requests per stage).
[[maybe_unused]] int encode_operand_map(CUtensorMap* map, const void* image, int64_t n, int kpad, int box_rows,
                       int box_kgroups = 0) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SJB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (box_rows % 32) return fail(SJB_E_INVALID, "box rows %d not a multiple of 32", box_rows);
  const int64_t rows = sjb::round_up(n, 2 * sjb::kTileRows);
  const cuuint64_t kgroups = (cuuint64_t)kpad / 8;
  const cuuint64_t dims[3] = {256, (cuuint64_t)sjb::kTileRows / 32,
                              kgroups * (cuuint64_t)(rows / sjb::kTileRows)};
  const cuuint64_t strides[2] = {512, (cuuint64_t)sjb::kTileRows * 16};
  const cuuint32_t box[3] = {256, (cuuint32_t)box_rows / 32,
                             (cuuint32_t)(box_kgroups > 0 ? box_kgroups : (int)kgroups)};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(image), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SJB_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SJB_OK;
}

// fp32 canonical rows f32[n][dim] (dim % 4 == 0) as a 2-D tensor; box =
// 32 elements x 256 rows = one K chunk of a tile, 128 B swizzle.
int encode_rows_map(CUtensorMap* map, const float* rows, int64_t n, int dim) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SJB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)dim, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)dim * 4};
  const cuuint32_t box[2] = {(cuuint32_t)sjb::wide::kRcKC, (cuuint32_t)sjb::kTileRows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(rows), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SJB_E_CUDA, "cuTensorMapEncodeTiled (rows) failed (%d)", (int)r);
  return SJB_OK;
}

#if SJB_AB_KERNELS
// fp32 rows f32[n][dim] (dim % 4 == 0, dim <= 256) for tile::gather4: box =
// one whole row, no swizzle (recheck_rows_kernel, A/B).
int encode_gather_rows_map(CUtensorMap* map, const float* rows, int64_t n, int dim) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SJB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)dim, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)dim * 4};
  const cuuint32_t box[2] = {(cuuint32_t)dim, 1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(rows), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SJB_E_CUDA, "cuTensorMapEncodeTiled (gather rows) failed (%d)", (int)r);
  return SJB_OK;
}
#endif

#if SJB_AB_KERNELS
template <int KS>
int launch_pair_ks(const sjb::pair::Params& pp, int grid, uint32_t smem, cudaStream_t st) {
  if (int rc = set_smem_attr((const void*)sjb::pair::filter_kernel<KS>, (int)smem)) return rc;
  sjb::pair::filter_kernel<KS><<<grid, sjb::pair::kThreads, smem, st>>>(pp);
  SJB_CK_LAUNCH("pair_filter");
  return SJB_OK;
}

int launch_pair_filter(const sjb::pair::Params& pp, int grid, uint32_t smem, cudaStream_t st) {
  switch (pp.kpad / 16) {
    case 1: return launch_pair_ks<1>(pp, grid, smem, st);
    case 2: return launch_pair_ks<2>(pp, grid, smem, st);
    case 3: return launch_pair_ks<3>(pp, grid, smem, st);
    case 4: return launch_pair_ks<4>(pp, grid, smem, st);
    case 5: return launch_pair_ks<5>(pp, grid, smem, st);
    case 6: return launch_pair_ks<6>(pp, grid, smem, st);
    case 7: return launch_pair_ks<7>(pp, grid, smem, st);
    case 8: return launch_pair_ks<8>(pp, grid, smem, st);
    default: return fail(SJB_E_UNSUPPORTED, "kpad %d", pp.kpad);
  }
}
#endif

int launch_join_filter(const sjb::JoinParams& jp, int grid, uint32_t smem, cudaStream_t st) {
  switch (jp.kpad / 16) {
    case 1: return launch_filter_ks<1>(jp, grid, smem, st);
    case 2: return launch_filter_ks<2>(jp, grid, smem, st);
    case 3: return launch_filter_ks<3>(jp, grid, smem, st);
    case 4: return launch_filter_ks<4>(jp, grid, smem, st);
    case 5: return launch_filter_ks<5>(jp, grid, smem, st);
    case 6: return launch_filter_ks<6>(jp, grid, smem, st);
    case 7: return launch_filter_ks<7>(jp, grid, smem, st);
    case 8: return launch_filter_ks<8>(jp, grid, smem, st);
    default: return fail(SJB_E_UNSUPPORTED, "kpad %d", jp.kpad);
  }
}

}  // namespace

namespace sjb {

// Publishes sjb_join_info into device memory.
__global__ void join_finalize_kernel(const unsigned long long* __restrict__ cta_count, int grid,
                                     uint64_t seg_cap, const uint64_t* __restrict__ rowoff,
                                     int64_t n_left, int64_t out_cap, int64_t* __restrict__ info) {
  __shared__ unsigned long long s_sum, s_max;
  if (threadIdx.x == 0) {
    s_sum = 0;
    s_max = 0;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < grid; c += blockDim.x) {
    atomicAdd(&s_sum, cta_count[c]);
    atomicMax(&s_max, cta_count[c]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t matches = n_left > 0 ? (int64_t)rowoff[n_left] : 0;
    const bool ovf = s_max > seg_cap || matches > out_cap;
    info[0] = matches;
    info[1] = (int64_t)s_sum;
    info[2] = (int64_t)(s_max * (unsigned long long)grid);
    reinterpret_cast<int32_t*>(info + 3)[0] = ovf ? 1 : 0;
    reinterpret_cast<int32_t*>(info + 3)[1] = grid;
  }
}

// Output gate (flag[1]): scatter/sort run only if the match count fits.
__global__ void gate_kernel(const uint64_t* __restrict__ rowoff, int64_t n_left, int64_t out_cap,
                            unsigned int* __restrict__ flag) {
  flag[1] = (n_left > 0 && (int64_t)rowoff[n_left] <= out_cap) ? 1u : 0u;
}

}  // namespace sjb

extern "C" {

int sjb_version(void) { return 1; }

// Diagnostics of the cluster-blocked dense recheck (built with
// -DSJB_BLK_STATS=1; otherwise returns SJB_E_UNSUPPORTED): copies the 16
// counters and zeroes them.
int sjb_debug_blk_stats(int64_t* out16) {
#if SJB_BLK_STATS
  unsigned long long h[16];
  SJB_CK(cudaMemcpyFromSymbol(h, sjb::g_blk_stats, sizeof(h)));
  for (int k = 0; k < 16; k++) out16[k] = (int64_t)h[k];
  memset(h, 0, sizeof(h));
  SJB_CK(cudaMemcpyToSymbol(sjb::g_blk_stats, h, sizeof(h)));
  return SJB_OK;
#else
  (void)out16;
  return fail(SJB_E_UNSUPPORTED, "built without SJB_BLK_STATS");
#endif
}

int64_t sjb_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* sjb_last_error(void) { return g_err.c_str(); }

int sjb_sm_count(int device) {
  static int cache[64] = {0};
  if (device >= 0 && device < 64 && cache[device]) return cache[device];
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  if (device >= 0 && device < 64) cache[device] = v;
  return v;
}

int64_t sjb_kpad(int64_t dim) {
  // <= 128: resident-R kernels, one UMMA k-step per 16; wider: K-streaming
  // kernel, 64-element chunks
  const int64_t d = dim < 1 ? 1 : dim;
  return d <= 128 ? sjb::round_up(d, 16) : sjb::round_up(d, sjb::wide::kKChunk);
}

int64_t sjb_operand_elems(int64_t n, int64_t dim) {
  // 512-row padding: the CTA-pair filter reads R blocks of two 256-row tiles
  return sjb::round_up(n < 0 ? 0 : n, 2 * sjb::kTileRows) * sjb_kpad(dim);
}

float sjb_default_band(int64_t dim) {
  // 16-bit operands: |op(x) - x| <= u|x| + 2^-25 per component (u = 2^-8 for
  // bf16 at kpad <= 128, 2^-11 for fp16 above; the 2^-25 covers fp16
  // subnormals and over-covers bf16's), so ||e_x|| <= e = u + 2^-25 sqrt(dim)
  // for a unit row, and by Cauchy-Schwarz |approx - exact| <= 2e(1 + 1e-6) +
  // e^2; plus fp32 accumulation error of both the tensor-core sum and the
  // canonical sequential sum (<= 2 * dim * 2^-24 each, generous).
  const double u = sjb::op_is_bf16((int)sjb_kpad(dim)) ? 1.0 / 256.0 : 1.0 / 2048.0;
  const double e = u + 2.98023223876953125e-08 * sqrt((double)dim);
  const double b = 2 * e * (1 + 1e-6) + e * e + 4.0 * (double)dim * 5.9604644775390625e-08 + 1e-6;
  return (float)b;
}

float sjb_accum_slack(int64_t dim) {
  // fp32 accumulation error of the tensor-core and canonical sums (as in
  // sjb_default_band) + 2e-6 for the fp32 evaluation of the per-row cutoff
  return (float)(4.0 * (double)dim * 5.9604644775390625e-08 + 2e-6);
}

int64_t sjb_tile_count(int64_t n) {
  return sjb::round_up(n < 0 ? 0 : n, 2 * sjb::kTileRows) / sjb::kTileRows;
}

static int normalize_impl(const float* d_in, const int64_t* d_gather, int64_t n, int64_t dim,
                          float* d_out32, void* d_out16, unsigned long long* d_repaired,
                          float* d_row_err, float* d_tile_err, void* stream) {
  if (n < 0 || dim < 1)
    return fail(SJB_E_INVALID, "bad shape n=%lld dim=%lld", (long long)n, (long long)dim);
  const int kpad = (int)sjb_kpad(dim);
  const int64_t tiles = d_out16 ? sjb_operand_elems(n, dim) / (kpad * (int64_t)sjb::kTileRows)
                                : sjb::ceil_div(n, sjb::kTileRows);
  if (tiles == 0) return SJB_OK;
  if (d_gather == nullptr && (dim & 3) == 0 && kpad <= 128 && ((uintptr_t)d_in & 15) == 0 &&
      ((uintptr_t)d_out32 & 15) == 0 && getenv("SJB_PREP_STAGED") == nullptr) {
    // pipelined kernel: per-warp 32-row slabs, double-buffered (8 warps per SM;
    // SJB_PREP_BUFS=1: one buffer, 16 warps)
    int dev = 0;
    cudaGetDevice(&dev);
    const char* pb = getenv("SJB_PREP_BUFS");
    const int nbuf = pb != nullptr && atoi(pb) == 1 ? 1 : 2;
    const int warps = sjb::pipe_warps((int)dim, nbuf, 210 * 1024);
    const int smem = sjb::pipe_smem_bytes((int)dim, nbuf, warps);
    if (int rc = set_smem_attr((const void*)sjb::normalize_pipe_kernel, smem)) return rc;
    auto st = as_stream(stream);
    const bool errs = d_out16 != nullptr && d_row_err != nullptr;
    if (errs && d_tile_err != nullptr) {
      cudaError_t e = cudaMemsetAsync(d_tile_err, 0, (size_t)tiles * 4, st);
      if (e != cudaSuccess) return fail(SJB_E_CUDA, "memset tile_err: %s", cudaGetErrorString(e));
    }
    const int64_t n_slabs = tiles * (sjb::kTileRows / sjb::kPipeSlab);
    const int64_t grid = sjb::mn<int64_t>(sjb::ceil_div(n_slabs, (int64_t)warps),
                                          (int64_t)sjb_sm_count(dev));
    sjb::normalize_pipe_kernel<<<(unsigned)grid, warps * 32, smem, st>>>(
        d_in, n, n_slabs, (int)dim, kpad, nbuf, d_out32, reinterpret_cast<sjb::op16_t*>(d_out16),
        d_repaired, errs ? d_row_err : nullptr,
        errs ? reinterpret_cast<unsigned*>(d_tile_err) : nullptr);
    SJB_CK_LAUNCH("normalize_pipe");
    return SJB_OK;
  }
  const int sub = prep_sub_rows(dim);
  const int smem = sub * (int)(dim | 1) * 4;
  if (int rc = set_smem_attr((const void*)sjb::normalize_cast_kernel, smem)) return rc;
  sjb::normalize_cast_kernel<<<(unsigned)tiles, sjb::kPrepThreads, smem, as_stream(stream)>>>(
      d_in, d_gather, n, (int)dim, kpad, sub, d_out32, reinterpret_cast<sjb::op16_t*>(d_out16),
      d_repaired, 1, d_out16 ? d_row_err : nullptr, d_out16 ? d_tile_err : nullptr);
  SJB_CK_LAUNCH("normalize_cast");
  return SJB_OK;
}

int sjb_normalize_rows(const float* d_in, int64_t n, int64_t dim, float* d_out32, void* d_out16,
                       unsigned long long* d_repaired, float* d_row_err, float* d_tile_err,
                       void* stream) {
  return normalize_impl(d_in, nullptr, n, dim, d_out32, d_out16, d_repaired, d_row_err,
                        d_tile_err, stream);
}

int sjb_gather_normalize_rows(const float* d_table, const int64_t* d_index, int64_t n,
                              int64_t dim, float* d_out32, void* d_out16,
                              unsigned long long* d_repaired, float* d_row_err,
                              float* d_tile_err, void* stream) {
  if (!d_index) return fail(SJB_E_INVALID, "null index");
  return normalize_impl(d_table, d_index, n, dim, d_out32, d_out16, d_repaired, d_row_err,
                        d_tile_err, stream);
}

int sjb_prepare_bf16(const void* d_in, int64_t n, int64_t dim, float* d_out32, void* d_out16,
                     float* d_inv_norm, unsigned long long* d_repaired, void* stream) {
  if (n < 0 || dim < 1 || !d_out32 || !d_out16 || !d_inv_norm)
    return fail(SJB_E_INVALID, "bad bf16 prep arguments");
  const int kpad = (int)sjb_kpad(dim);
  if (kpad <= 128) return fail(SJB_E_UNSUPPORTED, "sjb_prepare_bf16 is for dim > 128");
  const int64_t tiles = sjb_operand_elems(n, dim) / (kpad * (int64_t)sjb::kTileRows);
  if (tiles == 0) return SJB_OK;
  const int smem = sjb::kWideRows * (int)(dim | 1) * 4;
  if (int rc = set_smem_attr((const void*)sjb::prepare_bf16_kernel, smem)) return rc;
  sjb::prepare_bf16_kernel<<<(unsigned)tiles, sjb::kPrepThreads, smem, as_stream(stream)>>>(
      reinterpret_cast<const uint16_t*>(d_in), n, (int)dim, kpad, d_out32,
      reinterpret_cast<sjb::op16_t*>(d_out16), d_inv_norm, d_repaired);
  SJB_CK_LAUNCH("prepare_bf16");
  return SJB_OK;
}

int sjb_ab_kernels(void) { return SJB_AB_KERNELS; }

float sjb_raw_band(int64_t dim) {
  // exact bf16 products: fp32 accumulation of the tensor-core and canonical
  // sums (<= 2 dim 2^-24 each, generous), the canonical rows' and the inverse
  // norms' roundings and the two epilogue products (8 u), + 2e-6 for the fp32
  // evaluation of the cutoffs
  return (float)(4.0 * (double)dim * 5.9604644775390625e-08 + 8 * 5.9604644775390625e-08 + 2e-6);
}

int sjb_cast_rows(const float* d_in, int64_t n, int64_t dim, void* d_out16, void* stream) {
  if (n < 0 || dim < 1 || d_out16 == nullptr) return fail(SJB_E_INVALID, "bad cast arguments");
  const int kpad = (int)sjb_kpad(dim);
  const int64_t tiles = sjb_operand_elems(n, dim) / (kpad * (int64_t)sjb::kTileRows);
  if (tiles == 0) return SJB_OK;
  const int sub = prep_sub_rows(dim);
  const int smem = sub * (int)(dim | 1) * 4;
  if (int rc = set_smem_attr((const void*)sjb::normalize_cast_kernel, smem)) return rc;
  sjb::normalize_cast_kernel<<<(unsigned)tiles, sjb::kPrepThreads, smem, as_stream(stream)>>>(
      d_in, nullptr, n, (int)dim, kpad, sub, nullptr, reinterpret_cast<sjb::op16_t*>(d_out16),
      nullptr, 0, nullptr, nullptr);
  SJB_CK_LAUNCH("cast_rows");
  return SJB_OK;
}

int sjb_row_norms(const float* d_m, int64_t n, int64_t dim, float* d_out, void* stream) {
  if (n <= 0) return SJB_OK;
  sjb::row_norms_kernel<<<(unsigned)sjb::ceil_div(n, 256), 256, 0, as_stream(stream)>>>(
      d_m, n, (int)dim, d_out);
  SJB_CK_LAUNCH("row_norms");
  return SJB_OK;
}

int sjb_fnv1a64_many(const uint8_t* d_bytes, const int64_t* d_offs, int64_t n, uint64_t xor_seed,
                     uint64_t* d_out, void* stream) {
  if (n <= 0) return SJB_OK;
  sjb::fnv1a64_kernel<<<(unsigned)sjb::ceil_div(n, 256), 256, 0, as_stream(stream)>>>(
      d_bytes, d_offs, n, xor_seed, d_out);
  SJB_CK_LAUNCH("fnv1a64");
  return SJB_OK;
}

int sjb_synthetic_fill_many(const uint64_t* d_seeds, int64_t n, int64_t dim, float* d_out32,
                            void* d_out16, float* d_row_err, float* d_tile_err, void* stream) {
  if (n < 0 || dim < 1) return fail(SJB_E_INVALID, "bad shape");
  const int kpad = (int)sjb_kpad(dim);
  const int64_t tiles = d_out16 ? sjb_operand_elems(n, dim) / (kpad * (int64_t)sjb::kTileRows)
                                : sjb::ceil_div(n, sjb::kTileRows);
  if (tiles == 0) return SJB_OK;
  const int sub = prep_sub_rows(dim);
  const int smem = sub * (int)(dim | 1) * 4;
  if (int rc = set_smem_attr((const void*)sjb::synthetic_fill_kernel, smem)) return rc;
  sjb::synthetic_fill_kernel<<<(unsigned)tiles, sjb::kPrepThreads, smem, as_stream(stream)>>>(
      d_seeds, n, (int)dim, kpad, sub, d_out32, reinterpret_cast<sjb::op16_t*>(d_out16),
      d_out16 ? d_row_err : nullptr, d_out16 ? d_tile_err : nullptr);
  SJB_CK_LAUNCH("synthetic_fill");
  return SJB_OK;
}

int sjb_subword_embed(const uint8_t* d_bytes, const int64_t* d_offs, int64_t n,
                      const float* d_table, int64_t n_buckets, int64_t dim, int minn, int maxn,
                      int normalize, float* d_out32, void* d_out16,
                      unsigned long long* d_repaired, float* d_row_err, float* d_tile_err,
                      void* stream) {
  if (n < 0 || dim < 1 || n_buckets < 1 || minn < 1 || maxn < minn)
    return fail(SJB_E_INVALID, "bad subword arguments");
  const int kpad = (int)sjb_kpad(dim);
  const int64_t tiles = d_out16 ? sjb_operand_elems(n, dim) / (kpad * (int64_t)sjb::kTileRows)
                                : sjb::ceil_div(n, sjb::kTileRows);
  if (tiles == 0) return SJB_OK;
  const bool vec = (dim & 3) == 0 && dim <= 256 && ((uintptr_t)d_table & 15) == 0 &&
                   ((uintptr_t)d_out32 & 15) == 0 && getenv("SJB_SUBWORD_FUSED") == nullptr;
  if (vec) {
    // gather pass (mean rows into out32), then normalise-and-cast in place
    if (n > 0) {
      const uint64_t nb = (uint64_t)n_buckets, magic = ~0ULL / nb;
      int dev = 0;
      cudaGetDevice(&dev);
      const int64_t want = sjb::ceil_div(n, sjb::kGatherThreads / 32);
      auto st = as_stream(stream);
      // items in flight per warp (KU) against warps per SM (registers): an
      // A/B switch, SJB_SUBWORD_KU = 8 (4 CTAs/SM), 12 (3), 16 or 24 (2)
      // measured at cfg3 (200k strings, 2M x 100 table): KU 2: see DESIGN,
      // 4: 0.40 ms, 6: 0.45, 8: 0.48, 12: 0.56, 16: 0.75, 24: 0.80 -- warps
      // in flight beat items in flight per warp
      const char* ke = getenv("SJB_SUBWORD_KU");
      const int ku = ke ? atoi(ke) : 4;
      const int per_sm = ku <= 2 ? 8 : (ku <= 4 ? 6 : (ku <= 6 ? 5 : (ku <= 8 ? 4 : (ku <= 12 ? 3 : 2))));
      const int grid = (int)sjb::mn<int64_t>(want, (int64_t)sjb_sm_count(dev) * per_sm);
#define SJB_GATHER(V, KU, MB)                                                          \
  sjb::subword_gather_kernel<V, KU, MB><<<grid, sjb::kGatherThreads, 0, st>>>(          \
      d_bytes, d_offs, n, d_table, nb, magic, (int)dim, minn, maxn, d_out32)
      if (dim > 128) SJB_GATHER(2, 4, 3);
      else if (ku <= 2) SJB_GATHER(1, 2, 8);
      else if (ku <= 4) SJB_GATHER(1, 4, 6);
      else if (ku <= 6) SJB_GATHER(1, 6, 5);
      else if (ku <= 8) SJB_GATHER(1, 8, 4);
      else if (ku <= 12) SJB_GATHER(1, 12, 3);
      else if (ku <= 16) SJB_GATHER(1, 16, 2);
      else SJB_GATHER(1, 24, 2);
#undef SJB_GATHER
      SJB_CK_LAUNCH("subword_gather");
    }
    if (!normalize) return SJB_OK;
    return normalize_impl(d_out32, nullptr, n, dim, d_out32, d_out16, d_repaired,
                          d_out16 ? d_row_err : nullptr, d_out16 ? d_tile_err : nullptr, stream);
  }
  // gather-latency-bound: smaller staging sub-tiles fit twice the warps per SM
  const int sub = prep_sub_rows(dim) > 64 ? 64 : prep_sub_rows(dim);
  const int smem = sub * (int)(dim | 1) * 4;
  if (int rc = set_smem_attr((const void*)sjb::subword_embed_kernel, smem)) return rc;
  sjb::subword_embed_kernel<<<(unsigned)tiles, sjb::kPrepThreads, smem, as_stream(stream)>>>(
      d_bytes, d_offs, n, d_table, n_buckets, (int)dim, kpad, sub, minn, maxn, normalize, d_out32,
      normalize ? reinterpret_cast<sjb::op16_t*>(d_out16) : nullptr, d_repaired,
      normalize && d_out16 ? d_row_err : nullptr, normalize && d_out16 ? d_tile_err : nullptr);
  SJB_CK_LAUNCH("subword_embed");
  return SJB_OK;
}

int64_t sjb_join_workspace_bytes(const sjb_join_args* args) {
  if (!args) return -1;
  JoinPlan pl;
  int grid = 1;
  int64_t tstride = 0;
  if (args->n_left > 0 && args->n_right > 0) {
    if (make_plan(args, &pl) != SJB_OK) return -1;
    grid = pl.grid;
    tstride = pl.tile_stride;
  }
  return (int64_t)join_ws_layout(args, grid, tstride).total;
}

}  // extern "C"

namespace {

// One join's plan and workspace views (shared by the begin / filter-range /
// finish steps, which must all see the same args and workspace).
struct JoinCtx {
  JoinPlan pl;
  uint64_t* cand;
  uint32_t* sims_bits;
  unsigned long long* cta;
  uint32_t* rowcount;
  uint64_t *rowoff, *cursor, *keys, *bsums;
  uint32_t* bigrows;
  unsigned int* nbig;
  uint32_t* tile_off;
  uint64_t* ncand;  // dense recheck: number of grouped candidates
  unsigned int* work;  // wide group recheck: dynamic item counter
  uint32_t* sig;       // dense recheck: row signatures (smallest right offset)
  uint64_t* desc;      // dense recheck: blocks (start | rows << 32)
  uint32_t* ccnt;      // dense recheck: candidates per row
  bool empty;  // n_left == 0 or n_right == 0
  uint32_t* pend;
  uint32_t* pend_count;
};

int join_ctx(const sjb_join_args* args, void* d_workspace, int64_t workspace_bytes, JoinCtx* c) {
  if (!args) return fail(SJB_E_INVALID, "null args");
  const int64_t nl = args->n_left, nr = args->n_right;
  if (nl < 0 || nr < 0 || args->dim < 1) return fail(SJB_E_INVALID, "bad shape");
  if (nl >= (int64_t(1) << 32) || nr >= (int64_t(1) << 32))
    return fail(SJB_E_UNSUPPORTED, "relations are limited to 2^32 rows per join");
  c->empty = nl == 0 || nr == 0;
  if (c->empty) return SJB_OK;
  if (int rc = make_plan(args, &c->pl)) return rc;
  const JoinPlan& pl = c->pl;
  const JoinWs w = join_ws_layout(args, pl.grid, pl.tile_stride);
  if ((int64_t)w.total > workspace_bytes)
    return fail(SJB_E_INVALID, "workspace %lld B < required %lld B", (long long)workspace_bytes,
                (long long)w.total);
  if (pl.seg_cap < 1)
    return fail(SJB_E_INVALID, "cand_cap %lld < grid %d", (long long)args->cand_cap, pl.grid);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_workspace);
  c->cand = reinterpret_cast<uint64_t*>(ws + w.cand);
  c->sims_bits = reinterpret_cast<uint32_t*>(ws + w.sims);
  c->cta = reinterpret_cast<unsigned long long*>(ws + w.cta);
  c->rowcount = reinterpret_cast<uint32_t*>(ws + w.rowcount);
  c->rowoff = reinterpret_cast<uint64_t*>(ws + w.rowoff);
  c->cursor = reinterpret_cast<uint64_t*>(ws + w.cursor);
  c->keys = reinterpret_cast<uint64_t*>(ws + w.keys);
  c->bsums = reinterpret_cast<uint64_t*>(ws + w.bsums);
  c->bigrows = reinterpret_cast<uint32_t*>(ws + w.bigrows);
  c->nbig = reinterpret_cast<unsigned int*>(ws + w.nbig);
  c->tile_off = reinterpret_cast<uint32_t*>(ws + w.tiles);
  c->ncand = reinterpret_cast<uint64_t*>(ws + w.ncand);
  c->work = reinterpret_cast<unsigned int*>(ws + w.work);
  c->sig = reinterpret_cast<uint32_t*>(ws + w.sig);
  c->desc = reinterpret_cast<uint64_t*>(ws + w.desc);
  c->ccnt = reinterpret_cast<uint32_t*>(ws + w.ccnt);
  c->pend = reinterpret_cast<uint32_t*>(ws + w.pend);
  c->pend_count = reinterpret_cast<uint32_t*>(ws + w.pendn);
  return SJB_OK;
}

bool fused_recheck(const JoinPlan& pl) {
  return pl.wide ? pl.wide_fused : !pl.defer;
}

int join_begin(const sjb_join_args* args, const JoinCtx& c, cudaStream_t st) {
  const JoinPlan& pl = c.pl;
  SJB_CK(cudaMemsetAsync(c.rowcount, 0, (size_t)args->n_left * 4, st));
  SJB_CK(cudaMemsetAsync(c.nbig, 0, 16, st));
  SJB_CK(cudaMemsetAsync(c.cta, 0, (size_t)pl.grid * 8, st));
  if (args->sims_mode == 1 && c.pend_count != nullptr)   // a filter may launch fewer CTAs than pl.grid
    SJB_CK(cudaMemsetAsync(c.pend_count, 0, (size_t)pl.grid * 4, st));
  // candidate slots start empty: the fused recheck waits for each slot's write
  if (fused_recheck(pl))
    SJB_CK(cudaMemsetAsync(c.cand, 0xFF, (size_t)pl.grid * pl.seg_cap * 8, st));
  return SJB_OK;
}

// Work items over S tiles [tb, te) (kernel tile units): the plan's chunking,
// narrowed when the range is short so every CTA still gets ~8 items.
void range_items(const JoinPlan& pl, int64_t tb, int64_t te, int* tpc, int64_t* items) {
  const int64_t range = te - tb;
  int64_t t = (int64_t)pl.n_ablk * range / (8LL * pl.grid);
  t = t < 1 ? 1 : (t > pl.tiles_per_chunk ? pl.tiles_per_chunk : t);
  *tpc = (int)t;
  *items = range <= 0 ? 0 : (int64_t)pl.n_ablk * sjb::ceil_div(range, t);
}

// Filter (+ recheck) S tiles [tile_begin, tile_end) of 256 rows, appending to
// the per-CTA candidate segments.
int join_filter(const float* d_l32, const void* d_l16, const float* d_r32, const void* d_r16,
                const sjb_join_args* args, const JoinCtx& c, int64_t tile_begin,
                int64_t tile_end, cudaStream_t st) {
  const JoinPlan& pl = c.pl;
  const int64_t nl = args->n_left, nr = args->n_right;
  const int64_t nt256 = sjb::ceil_div(nr, sjb::kTileRows);
  if (tile_begin < 0) tile_begin = 0;
  if (tile_end > nt256) tile_end = nt256;
  if (tile_end <= tile_begin) return SJB_OK;
  // kernel tile units: 256 rows, or 128 for the CTA-pair kernel
#if SJB_AB_KERNELS
  const int64_t unit = pl.pair ? sjb::kTileRows / sjb::pair::kUmmaN : 1;
#else
  const int64_t unit = 1;
#endif
  const int64_t tb = tile_begin * unit;
  const int64_t te = tile_end * unit > pl.n_btiles ? pl.n_btiles : tile_end * unit;
  int tpc = 0;
  int64_t items = 0;
  range_items(pl, tb, te, &tpc, &items);
  if (pl.pair) {
    // pair items cover pairs of CTAs; the plan's grid is 2 CTAs per item lane
    int64_t t = (int64_t)pl.n_ablk * (te - tb) / (8LL * (pl.grid / 2));
    tpc = (int)(t < 1 ? 1 : (t > pl.tiles_per_chunk ? pl.tiles_per_chunk : t));
    items = (int64_t)pl.n_ablk * sjb::ceil_div(te - tb, (int64_t)tpc);
  }

  sjb::JoinParams jp;
  jp.a16 = reinterpret_cast<const sjb::op16_t*>(d_l16);
  jp.b16 = reinterpret_cast<const sjb::op16_t*>(d_r16);
  jp.n_a = nl;
  jp.n_b = nr;
  jp.kpad = pl.kpad;
  jp.n_ablk = pl.n_ablk;
  jp.n_btiles = (int)te;
  jp.tiles_per_chunk = tpc;
  jp.tile_begin = (int)tb;
  jp.append = 1;
  jp.defer = pl.defer ? 1 : 0;
  jp.n_items = items;
  jp.stages = pl.stages;
  jp.a_bufs = pl.a_bufs;
  jp.a_tiles = pl.a_tiles;
  jp.ts = pl.ts ? 1 : 0;
  jp.cutoff = args->theta - args->band;
  const bool per_row = args->left_row_err != nullptr && args->right_tile_err != nullptr;
  jp.row_err = per_row ? args->left_row_err : nullptr;
  jp.tile_err = per_row ? args->right_tile_err : nullptr;
  jp.slack = sjb_accum_slack(args->dim);
  jp.cand = c.cand;
  jp.seg_cap = pl.seg_cap;
  jp.cta_count = c.cta;
  jp.l32 = d_l32;
  jp.r32 = d_r32;
  jp.dim = (int)args->dim;
  jp.theta = args->theta;
  jp.sims_bits = c.sims_bits;
  jp.rowcount = c.rowcount;
  {
    const char* dm = getenv("SJB_DEBUG_MODE");
    jp.debug_mode = dm ? atoi(dm) : 0;
  }
  if (args->ev_filter_begin)
    SJB_CK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(args->ev_filter_begin), st));
  if (pl.wide) {
    sjb::wide::Params wp;
    wp.a16 = jp.a16;
    wp.b16 = jp.b16;
    wp.n_a = nl;
    wp.n_b = nr;
    wp.kpad = pl.kpad;
    wp.n_ablk = pl.n_ablk;
    wp.n_btiles = jp.n_btiles;
    wp.tiles_per_chunk = tpc;
    wp.tile_begin = jp.tile_begin;
    wp.append = 1;
    wp.n_items = items;
    wp.stages = pl.stages;
    wp.cutoff = jp.cutoff;
    wp.row_err = jp.row_err;
    wp.tile_err = jp.tile_err;
    wp.slack = jp.slack;
    wp.cand = c.cand;
    wp.seg_cap = pl.seg_cap;
    wp.cta_count = c.cta;
    wp.l32 = d_l32;
    wp.r32 = d_r32;
    wp.dim = (int)args->dim;
    wp.theta = args->theta;
    wp.sims_bits = c.sims_bits;
    wp.rowcount = c.rowcount;
    wp.debug = jp.debug_mode;
    wp.tile_off = c.tile_off;
    wp.tile_stride = pl.tile_stride;
    wp.inv_a = args->left_inv_norm;
    wp.inv_b = args->right_inv_norm;
    wp.tol = args->sims_mode == 1 ? 1 : 0;
    wp.hi_cut = args->theta + args->band;
    wp.pend = c.pend;
    wp.pend_count = c.pend_count;
    if (wp.inv_a != nullptr) {   // raw operands: the uniform accumulation band only
      wp.row_err = nullptr;
      wp.tile_err = nullptr;
    }
    if (pl.wide_fused) {
#if SJB_AB_KERNELS
      if (int rc = set_smem_attr((const void*)sjb::wide::filter_kernel<true>, (int)pl.smem)) return rc;
      sjb::wide::filter_kernel<true>
          <<<pl.grid, sjb::wide::Cfg<true>::kThreads, pl.smem, st>>>(wp);
      SJB_CK_LAUNCH("wide_filter_fused");
#else
      return ab_missing("SJB_WIDE_RECHECK=fused");
#endif
    } else {
      // A/B (SJB_WIDE_PAIR=1, tolerance emission only): CTA pairs sharing
      // each S chunk by TMA multicast -- measured slower (cfg4 slice 33.8 vs
      // 31.1 ms: the coupled rings wait on the slower CTA's epilogue)
      const char* wpv = getenv("SJB_WIDE_PAIR");
      const bool wpair = wp.tol && (pl.grid % 2) == 0 && wpv && strcmp(wpv, "1") == 0;
      // Tensor sims on raw bf16 operands run on CTA pairs (sjb_join4.cu,
      // cta_group::2): by default 256 x 256 pair tiles with TWO accumulator
      // stages, so a tile's drain, normalisation and emission overlap the next
      // tile's MMAs (cfg4 slice: filter 22.0 -> 15.2 ms, tensor pipe 51 -> 97%
      // active).  SJB_WIDE_MMA2=0: the 1-CTA kernel of sjb_join3.cu (A/B);
      // =1 (A/B build): 256 x 512 pair tiles, one accumulator tile -- measured
      // no faster than the 1-CTA kernel (32.8 vs 31.0 ms).
      const char* m2v = getenv("SJB_WIDE_MMA2");
      const bool mma2_one = m2v != nullptr && strcmp(m2v, "1") == 0;
      const bool mma2_two_env = !mma2_one && !(m2v != nullptr && strcmp(m2v, "0") == 0);
      const bool mma2 = pl.wide_rows ||
                        (wp.tol && wp.inv_a != nullptr && (pl.grid % 2) == 0 && !wpair &&
                         (mma2_two_env || (mma2_one && (tb % 2) == 0)));
      if (mma2) {
#if !SJB_AB_KERNELS
        if (mma2_one && !pl.wide_rows) return ab_missing("SJB_WIDE_MMA2=1");
#endif
        const bool mma2_two = pl.wide_rows || mma2_two_env;
        sjb::wide2::Params q;
        q.tol = wp.tol;
        q.tile_off = c.tile_off;
        q.tile_stride = pl.tile_stride;
        if (int rc = encode_operand_map(&q.tmap_a, d_l16, nl, pl.kpad, 128, 8)) return rc;
        if (int rc = encode_operand_map(&q.tmap_b, d_r16, nr, pl.kpad, 128, 8)) return rc;
        q.n_a = nl;
        q.n_b = nr;
        q.kpad = pl.kpad;
        q.n_ablk = pl.n_ablk;
        // 512-row pair tiles (the image is padded); two-stage: the 256-row tiles themselves
        const int64_t pb = mma2_two ? tb : tb / 2, pe = mma2_two ? te : (te + 1) / 2;
        const int64_t tt = (int64_t)pl.n_ablk * (pe - pb) / (8LL * (pl.grid / 2));
        int tpc2 = (int)(tt < 1 ? 1 : (tt > 32 ? 32 : tt));
        if (pl.wide_rows) {
          // the per-CTA item offsets share the tile-offset rows of the workspace: coarser
          // items until a pair's items (+ the end offset) fit one row
          const int64_t np2 = pl.grid / 2;
          while (tpc2 < 32 &&
                 sjb::ceil_div((int64_t)pl.n_ablk * sjb::ceil_div(pe - pb, (int64_t)tpc2), np2) + 1 >
                     pl.tile_stride)
            tpc2 *= 2;
        }
        q.n_ptiles = (int)pe;
        q.tiles_per_chunk = tpc2;
        q.tile_begin = (int)pb;
        q.append = 1;
        q.n_items = (int64_t)pl.n_ablk * sjb::ceil_div(pe - pb, (int64_t)tpc2);
        q.stages = sjb::wide2::max_stages(mma2_two);
        q.bf16 = 1;
        q.cutoff = wp.cutoff;
        q.hi_cut = wp.hi_cut;
        q.cand = c.cand;
        q.seg_cap = pl.seg_cap;
        q.cta_count = c.cta;
        q.inv_a = wp.inv_a;
        q.inv_b = wp.inv_b;
        q.sims_bits = c.sims_bits;
        q.rowcount = c.rowcount;
        q.pend = c.pend;
        q.pend_count = c.pend_count;
        q.debug = jp.debug_mode;
        const uint32_t sm2 = sjb::wide2::smem_bytes(q.stages, mma2_two);
        if (mma2_two) {
          if (int rc = set_smem_attr((const void*)sjb::wide2::filter_kernel<true>, (int)sm2)) return rc;
          // the kernel is persistent with a static item -> pair map: every pair must be
          // resident at once.  A GPC with an odd number of free SMs strands one, so ask
          // how many 2-CTA clusters fit and launch no more (CTAs beyond them keep empty
          // candidate segments; the count is the same for every launch of a join)
          static int max_pairs[64] = {};
          const int dv = current_device();
          if (dv >= 0 && dv < 64 && max_pairs[dv] == 0) {
            cudaLaunchConfig_t oc = {};
            oc.gridDim = dim3((unsigned)pl.grid);
            oc.blockDim = dim3(sjb::wide2::kThreads);
            oc.dynamicSmemBytes = sm2;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, sjb::wide2::filter_kernel<true>, &oc) !=
                    cudaSuccess || nc <= 0) {
              (void)cudaGetLastError();
              nc = 1 << 20;   // unknown: do not limit
            }
            max_pairs[dv] = nc;
          }
          const int lim = (dv >= 0 && dv < 64) ? max_pairs[dv] : (1 << 20);
          const int g2 = 2 * (pl.grid / 2 < lim ? pl.grid / 2 : lim);
          sjb::wide2::filter_kernel<true><<<g2, sjb::wide2::kThreads, sm2, st>>>(q);
          if (pl.wide_rows && jp.debug_mode != 1) {
            // every candidate of this launch, work items in the filter's S-chunk-major order
            SJB_CK_LAUNCH("wide2_filter");
            SJB_CK(cudaMemsetAsync(c.work, 0, 4, st));
            const uint32_t rsm = sjb::wide::recheck_sorted_smem();
            if (int rc = set_smem_attr((const void*)sjb::wide::recheck_segments_sorted_kernel,
                                       (int)rsm))
              return rc;
            sjb::wide::recheck_segments_sorted_kernel<<<sjb_sm_count(current_device()),
                                                        sjb::wide::kPsWarps * 32, rsm, st>>>(
                c.cand, pl.seg_cap, c.cta, c.tile_off, pl.tile_stride, q.n_items, g2 / 2, c.work,
                d_l32, d_r32, (int)args->dim, args->theta, c.sims_bits, c.rowcount);
          }
        } else {
#if SJB_AB_KERNELS
          if (int rc = set_smem_attr((const void*)sjb::wide2::filter_kernel<false>, (int)sm2)) return rc;
          sjb::wide2::filter_kernel<false><<<pl.grid, sjb::wide2::kThreads, sm2, st>>>(q);
#endif
        }
        SJB_CK_LAUNCH("wide2_filter");
      } else if (wpair) {
#if !SJB_AB_KERNELS
        return ab_missing("SJB_WIDE_PAIR=1");
#else
        const void* fn = (const void*)sjb::wide::filter_kernel<false, true>;
        if (int rc = set_smem_attr(fn, (int)pl.smem)) return rc;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)pl.grid);
        cfg.blockDim = dim3(sjb::wide::Cfg<false>::kThreads);
        cfg.dynamicSmemBytes = pl.smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SJB_CK(cudaLaunchKernelEx(&cfg, sjb::wide::filter_kernel<false, true>, wp));
        SJB_CK_LAUNCH("wide_filter_pair");
#endif
      } else {
        if (int rc = set_smem_attr((const void*)sjb::wide::filter_kernel<false>, (int)pl.smem))
          return rc;
        sjb::wide::filter_kernel<false>
            <<<pl.grid, sjb::wide::Cfg<false>::kThreads, pl.smem, st>>>(wp);
        SJB_CK_LAUNCH("wide_filter");
      }
      if (pl.wide_rows) {
        // candidates only: join_finish groups them by left row and rechecks them there
      } else if (wp.tol && jp.debug_mode != 1) {
        // tolerance emission: only the band pairs need the canonical chain
        // rows staged through shared memory by whole warps (default; dim % 4 = 0 and
        // 16-byte aligned rows); SJB_PENDING=gather: the thread-per-pair gather (A/B)
        const char* pv = getenv("SJB_PENDING");
        const bool staged = (args->dim % 4) == 0 &&
                            ((reinterpret_cast<uintptr_t>(d_l32) | reinterpret_cast<uintptr_t>(d_r32)) & 15) == 0 &&
                            !(pv != nullptr && strcmp(pv, "gather") == 0);
        if (staged) {
          const uint32_t psm = sjb::wide::pending_staged_smem();
          if (int rc = set_smem_attr((const void*)sjb::wide::recheck_pending_staged_kernel, (int)psm))
            return rc;
          sjb::wide::recheck_pending_staged_kernel<<<sjb_sm_count(current_device()),
                                                     sjb::wide::kPsWarps * 32, psm, st>>>(
              c.cand, pl.seg_cap, c.pend, c.pend_count, c.cta, pl.grid, d_l32, d_r32,
              (int)args->dim, args->theta, c.sims_bits, c.rowcount);
        } else {
          sjb::wide::recheck_pending_kernel<<<sjb_sm_count(current_device()) * 8, 256, 0, st>>>(
              c.cand, pl.seg_cap, c.pend, c.pend_count, c.cta, pl.grid, d_l32, d_r32,
              (int)args->dim, args->theta, c.sims_bits, c.rowcount);
        }
        SJB_CK_LAUNCH("recheck_pending");
      } else if (jp.debug_mode != 1) {
        sjb::wide::RecheckParams rp;
        rp.cand = c.cand;
        rp.seg_cap = pl.seg_cap;
        rp.cta_count = c.cta;
        rp.tile_off = c.tile_off;
        rp.tile_stride = pl.tile_stride;
        rp.n_items = items;
        rp.n_ablk = pl.n_ablk;
        rp.n_btiles = jp.n_btiles;
        rp.tiles_per_chunk = tpc;
        rp.tile_begin = jp.tile_begin;
        rp.n_a = nl;
        rp.n_b = nr;
        rp.l32 = d_l32;
        rp.r32 = d_r32;
        rp.dim = (int)args->dim;
        rp.theta = args->theta;
        rp.sims_bits = c.sims_bits;
        rp.rowcount = c.rowcount;
        {
          const char* dm = getenv("SJB_WIDE_DIRECT_MAX");
          rp.direct_max = dm ? (uint32_t)atoi(dm) : (uint32_t)sjb::wide::kRcDirect;
        }
        if ((args->dim & 3) == 0) {
          sjb::wide::RecheckTmaParams tp;
          tp.b = rp;
          if (int rc = encode_rows_map(&tp.tmap_l, d_l32, nl, (int)args->dim)) return rc;
          if (int rc = encode_rows_map(&tp.tmap_r, d_r32, nr, (int)args->dim)) return rc;
          const char* wr = getenv("SJB_WIDE_RECHECK");
          if (wr != nullptr && strcmp(wr, "tile") == 0) {  // A/B: A restaged per tile
#if SJB_AB_KERNELS
            const int rs = (int)sjb::wide::recheck_tma_smem_bytes();
            if (int rc = set_smem_attr((const void*)sjb::wide::recheck_tma_kernel, rs)) return rc;
            sjb::wide::recheck_tma_kernel<<<pl.grid, sjb::wide::kRtThreads, rs, st>>>(tp);
#else
            return ab_missing("SJB_WIDE_RECHECK=tile");
#endif
          } else {
            const int rs = (int)sjb::wide::recheck_group_smem_bytes();
            if (int rc = set_smem_attr((const void*)sjb::wide::recheck_group_kernel, rs)) return rc;
            SJB_CK(cudaMemsetAsync(c.work, 0, 4, st));
            tp.b.work = c.work;
            tp.b.filter_grid = pl.grid;
            sjb::wide::recheck_group_kernel<<<pl.grid, sjb::wide::kRtThreads, rs, st>>>(tp);
          }
        } else {
          const int rs = (int)sjb::wide::recheck_smem_bytes();
          if (int rc = set_smem_attr((const void*)sjb::wide::recheck_generic_kernel, rs)) return rc;
          sjb::wide::recheck_generic_kernel<<<pl.grid, sjb::wide::kRcThreads, rs, st>>>(rp);
        }
        SJB_CK_LAUNCH("wide_recheck");
      }
    }
  } else if (pl.pair) {
#if SJB_AB_KERNELS
    sjb::pair::Params pp;
    pp.a16 = jp.a16;
    pp.b16 = jp.b16;
    pp.n_a = nl;
    pp.n_b = nr;
    pp.kpad = pl.kpad;
    pp.n_ablk = pl.n_ablk;
    pp.n_btiles = jp.n_btiles;
    pp.tiles_per_chunk = tpc;
    pp.tile_begin = jp.tile_begin;
    pp.append = 1;
    pp.n_items = items;
    pp.stages = pl.stages;
    pp.cutoff = jp.cutoff;
    pp.row_err = jp.row_err;
    pp.tile_err = jp.tile_err;
    pp.slack = jp.slack;
    pp.cand = c.cand;
    pp.seg_cap = pl.seg_cap;
    pp.cta_count = c.cta;
    pp.l32 = d_l32;
    pp.r32 = d_r32;
    pp.dim = (int)args->dim;
    pp.theta = args->theta;
    pp.sims_bits = c.sims_bits;
    pp.rowcount = c.rowcount;
    pp.debug_mode = jp.debug_mode;
    if (int rc = encode_operand_map(&pp.tmap_a, d_l16, nl, pl.kpad, sjb::pair::kARows)) return rc;
    if (int rc = encode_operand_map(&pp.tmap_b, d_r16, nr, pl.kpad, sjb::pair::kHalfN)) return rc;
    if (int rc = launch_pair_filter(pp, pl.grid, pl.smem, st)) return rc;
#else
    return ab_missing("SJB_FILTER=pair");
#endif
  } else {
    const int lg = args->launch_grid > 0 && args->launch_grid < pl.grid ? args->launch_grid
                                                                         : pl.grid;
    if (int rc = launch_join_filter(jp, lg, pl.smem, st)) return rc;
  }
  if (args->ev_filter_end)
    SJB_CK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(args->ev_filter_end), st));
  return SJB_OK;
}

// Row offsets, then bucket by left row and sort each row by right offset.
int join_finish(const float* d_l32, const float* d_r32, const sjb_join_args* args,
                const JoinCtx& c, uint64_t* d_lefts,
                uint64_t* d_rights, float* d_sims, int64_t* info, cudaStream_t st) {
  const JoinPlan& pl = c.pl;
  const int64_t nl = args->n_left;
  const uint64_t slots = (uint64_t)pl.grid * pl.seg_cap;
  uint64_t* keys = c.keys;
  if (pl.defer && use_rows_recheck(args, d_l32, d_r32) && dense_mode() == 0) {
    // dense (sjb_post.cu): count per row (+ signature); order the rows by
    // hashed signature and cut the order into blocks; lay the candidates out
    // in that order (each block contiguous, right offsets only); recheck the
    // blocks; match offsets; one pass to the MatchSet columns
    const int dev = current_device();
    const int sms = sjb_sm_count(dev);
    const int fg = grid_for((uint64_t)nl, 256, 8);
    SJB_CK(cudaMemsetAsync(c.sig, 0xFF, (size_t)nl * 4, st));
    SJB_CK(cudaMemsetAsync(c.ccnt, 0, (size_t)nl * 4, st));
    // chunks of 2048 candidates aggregated per row in shared memory; enough
    // CTAs per segment for kAggCtasPerSm per SM (SJB_AGG_CTAS overrides)
    const char* acv = getenv("SJB_AGG_CTAS");
    const int kAggCtasPerSm = acv ? std::max(1, atoi(acv)) : 16;
    const dim3 agrid((unsigned)std::max(1, kAggCtasPerSm * sms / pl.grid), (unsigned)pl.grid);
    sjb::count_rows_agg_kernel<<<agrid, sjb::kAggThreads, 0, st>>>(c.cand, pl.seg_cap, c.cta,
                                                                   c.ccnt, c.sig);
    SJB_CK_LAUNCH("count_rows_agg");
    // the order: hashed signature buckets (perm in bigrows), blocks in desc
    const int shift = 0;
    SJB_CK(cudaMemsetAsync(c.rowcount, 0, (size_t)nl * 4, st));
    sjb::sig_hist_kernel<<<fg, 256, 0, st>>>(c.sig, c.ccnt, nl, shift, c.rowcount);
    SJB_CK_LAUNCH("sig_hist");
    if (int rc = run_scan(c.rowcount, nl, c.cursor, nullptr, c.bsums, st)) return rc;
    sjb::sig_scatter_kernel<<<fg, 256, 0, st>>>(
        c.sig, c.ccnt, nl, shift, reinterpret_cast<unsigned long long*>(c.cursor), c.bigrows);
    SJB_CK_LAUNCH("sig_scatter");
    SJB_CK(cudaMemsetAsync(c.work, 0, 8, st));   // [0] block counter, [1] blocks
    sjb::sig_blocks_kernel<<<fg, 256, 0, st>>>(c.rowcount, c.cursor, nl, c.desc, c.work + 1);
    SJB_CK_LAUNCH("sig_blocks");
    // candidate offsets in the blocks' order (rowoff = poff), row starts in cursor
    sjb::perm_counts_kernel<<<fg, 256, 0, st>>>(c.bigrows, c.ccnt, nl, c.rowcount);
    SJB_CK_LAUNCH("perm_counts");
    if (int rc = run_scan(c.rowcount, nl, c.rowoff, nullptr, c.bsums, st)) return rc;
    sjb::perm_starts_kernel<<<fg, 256, 0, st>>>(c.bigrows, c.rowoff, nl, c.cursor);
    SJB_CK_LAUNCH("perm_starts");
    // right offsets grouped (u32, in the sims buffer: the filter wrote none)
    sjb::group_rows_agg_kernel<uint32_t><<<agrid, sjb::kAggThreads, 0, st>>>(
        c.cand, pl.seg_cap, c.cta, reinterpret_cast<unsigned long long*>(c.cursor), c.sims_bits);
    SJB_CK_LAUNCH("group_rows_agg");
    const int bsmem = sjb::blk_smem_bytes((int)args->dim);
    if (int rc = set_smem_attr((const void*)sjb::recheck_blocks_kernel, bsmem)) return rc;
    int per_sm = 0;
    SJB_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sjb::recheck_blocks_kernel,
                                                         sjb::kBlkThreads, bsmem));
    sjb::recheck_blocks_kernel<<<sms * std::min(2, std::max(1, per_sm)), sjb::kBlkThreads, bsmem,
                                 st>>>(c.sims_bits, c.rowoff, c.ccnt, c.keys, c.bigrows, c.desc,
                                       c.work + 1, d_l32, d_r32, (int)args->dim, args->theta,
                                       c.rowcount, c.work);
    SJB_CK_LAUNCH("recheck_blocks");
    // match offsets (row order) into `rowoff`; `cursor` holds the rows' candidate ends
    if (int rc = run_scan(c.rowcount, nl, c.rowoff, nullptr, c.bsums, st)) return rc;
    sjb::gate_kernel<<<1, 1, 0, st>>>(c.rowoff, nl, args->out_cap, c.nbig);
    SJB_CK_LAUNCH("gate");
    sjb::emit_sims_kernel<<<grid_for((uint64_t)nl * 32, 256, 8), 256, 0, st>>>(
        c.keys, c.cursor, c.ccnt, c.rowoff, nl, d_lefts, d_rights, d_sims, c.cand, c.bigrows,
        c.nbig, args->left_base);
    SJB_CK_LAUNCH("emit_sims");
    const int big_smem = sjb::kSortBigCap * 8;
    if (int rc = set_smem_attr((const void*)sjb::segsort_big_kernel, big_smem)) return rc;
    sjb::segsort_big_kernel<<<sms, sjb::kSortBigThreads, big_smem, st>>>(
        c.rowoff, c.cand, d_lefts, d_rights, d_sims, c.bigrows, c.nbig, args->left_base,
        args->n_right);
    SJB_CK_LAUNCH("segsort_big");
    sjb::join_finalize_kernel<<<1, 256, 0, st>>>(c.cta, pl.grid, pl.seg_cap, c.rowoff, nl,
                                                 args->out_cap, info);
    SJB_CK_LAUNCH("finalize");
    return SJB_OK;
  }
  if (pl.defer && use_rows_recheck(args, d_l32, d_r32)) {
#if !SJB_AB_KERNELS
    return ab_missing("SJB_DENSE_RECHECK=rows");
#else
    // dense: group the candidates by left row; one warp per row sorts its
    // right offsets, rechecks them with bulk-copied S rows and compacts the
    // matches in place; then the match offsets and one copy to the columns
    const dim3 sgrid(8, (unsigned)pl.grid);
    sjb::count_rows_kernel<<<sgrid, 256, 0, st>>>(c.cand, pl.seg_cap, c.cta, c.rowcount, nullptr);
    SJB_CK_LAUNCH("count_rows");
    if (int rc = run_scan(c.rowcount, nl, c.rowoff, c.cursor, c.bsums, st)) return rc;
    sjb::group_rows_kernel<<<sgrid, 256, 0, st>>>(c.cand, pl.seg_cap, c.cta,
                                                  reinterpret_cast<unsigned long long*>(c.cursor),
                                                  c.keys);
    SJB_CK_LAUNCH("group_rows");
    SJB_CK(cudaMemsetAsync(c.work, 0, 4, st));
    const int dev = current_device();
    // S rows by tile::gather4 tensor copies (4 rows per copy) unless the map
    // cannot be encoded or SJB_ROWS_G4=0 (per-lane 1-D copies, A/B)
    CUtensorMap rmap;
    const char* g4env = getenv("SJB_ROWS_G4");
    const bool g4 = !(g4env && strcmp(g4env, "0") == 0) &&
                    encode_gather_rows_map(&rmap, d_r32, args->n_right, (int)args->dim) == SJB_OK;
    if (!g4) memset(&rmap, 0, sizeof(rmap));
    const int per_warp = sjb::rows_warp_smem((int)args->dim, g4);
    const int nw = std::min(8, (kRowsSmemMax - 128) / per_warp);
    const void* fn = g4 ? (const void*)sjb::recheck_rows_kernel<true>
                        : (const void*)sjb::recheck_rows_kernel<false>;
    if (int rc = set_smem_attr(fn, nw * per_warp + 128)) return rc;
    if (g4)
      sjb::recheck_rows_kernel<true><<<sjb_sm_count(dev), nw * 32, nw * per_warp + 128, st>>>(
          c.keys, c.rowoff, nl, d_l32, d_r32, (int)args->dim, args->theta, c.rowcount, c.work,
          rmap);
    else
      sjb::recheck_rows_kernel<false><<<sjb_sm_count(dev), nw * 32, nw * per_warp + 128, st>>>(
          c.keys, c.rowoff, nl, d_l32, d_r32, (int)args->dim, args->theta, c.rowcount, c.work,
          rmap);
    SJB_CK_LAUNCH("recheck_rows");
    // match offsets into `cursor`; `rowoff` keeps the candidate offsets
    if (int rc = run_scan(c.rowcount, nl, c.cursor, nullptr, c.bsums, st)) return rc;
    sjb::gate_kernel<<<1, 1, 0, st>>>(c.cursor, nl, args->out_cap, c.nbig);
    SJB_CK_LAUNCH("gate");
    sjb::emit_rows_kernel<<<grid_for((uint64_t)nl * 32, 256, 8), 256, 0, st>>>(
        c.keys, c.rowoff, c.cursor, nl, d_lefts, d_rights, d_sims, c.cand, c.bigrows, c.nbig,
        args->left_base);
    SJB_CK_LAUNCH("emit_rows");
    const int big_smem = sjb::kSortBigCap * 8;
    if (int rc = set_smem_attr((const void*)sjb::segsort_big_kernel, big_smem)) return rc;
    sjb::segsort_big_kernel<<<sjb_sm_count(dev), sjb::kSortBigThreads, big_smem, st>>>(
        c.cursor, c.cand, d_lefts, d_rights, d_sims, c.bigrows, c.nbig, args->left_base,
        args->n_right);
    SJB_CK_LAUNCH("segsort_big");
    sjb::join_finalize_kernel<<<1, 256, 0, st>>>(c.cta, pl.grid, pl.seg_cap, c.cursor, nl,
                                                 args->out_cap, info);
    SJB_CK_LAUNCH("finalize");
    return SJB_OK;
#endif
  }
  if (pl.defer) {
    // dense: group the candidates by left row, recheck them row-grouped,
    // then compact the matches by row (the segment buffer is free by then)
    const dim3 sgrid(8, (unsigned)pl.grid);
    sjb::count_rows_kernel<<<sgrid, 256, 0, st>>>(c.cand, pl.seg_cap, c.cta, c.rowcount, nullptr);
    SJB_CK_LAUNCH("count_rows");
    if (int rc = run_scan(c.rowcount, nl, c.rowoff, c.cursor, c.bsums, st)) return rc;
    SJB_CK(cudaMemcpyAsync(c.ncand, c.rowoff + nl, 8, cudaMemcpyDeviceToDevice, st));
    sjb::group_rows_kernel<<<sgrid, 256, 0, st>>>(c.cand, pl.seg_cap, c.cta,
                                                  reinterpret_cast<unsigned long long*>(c.cursor),
                                                  c.keys);
    SJB_CK_LAUNCH("group_rows");
    SJB_CK(cudaMemsetAsync(c.rowcount, 0, (size_t)nl * 4, st));
    const unsigned flat = (unsigned)sjb_sm_count(current_device()) * 8;
    sjb::recheck_grouped_kernel<<<flat, 256, 0, st>>>(c.keys, c.ncand, d_l32, d_r32,
                                                      (int)args->dim, args->theta, c.sims_bits,
                                                      c.rowcount);
    SJB_CK_LAUNCH("recheck_grouped");
    if (int rc = run_scan(c.rowcount, nl, c.rowoff, c.cursor, c.bsums, st)) return rc;
    sjb::gate_kernel<<<1, 1, 0, st>>>(c.rowoff, nl, args->out_cap, c.nbig);
    SJB_CK_LAUNCH("gate");
    keys = c.cand;
    sjb::compact_rows_kernel<<<flat, 256, 0, st>>>(
        c.keys, c.sims_bits, c.ncand, reinterpret_cast<unsigned long long*>(c.cursor), keys,
        c.nbig);
    SJB_CK_LAUNCH("compact_rows");
  } else {
    if (int rc = run_scan(c.rowcount, nl, c.rowoff, c.cursor, c.bsums, st)) return rc;
    sjb::gate_kernel<<<1, 1, 0, st>>>(c.rowoff, nl, args->out_cap, c.nbig);
    SJB_CK_LAUNCH("gate");
    sjb::scatter_kernel<<<grid_for(slots, 256, 8), 256, 0, st>>>(
        c.cand, pl.seg_cap, c.cta, pl.grid, c.sims_bits,
        reinterpret_cast<unsigned long long*>(c.cursor), c.keys, c.nbig);
    SJB_CK_LAUNCH("scatter");
  }
  sjb::segsort_small_kernel<<<grid_for((uint64_t)nl * 32, sjb::kSortSmallThreads, 16),
                              sjb::kSortSmallThreads, 0, st>>>(
      c.rowoff, nl, keys, d_lefts, d_rights, d_sims, c.bigrows, c.nbig, args->left_base);
  SJB_CK_LAUNCH("segsort_small");
  const int big_smem = sjb::kSortBigCap * 8;
  if (int rc = set_smem_attr((const void*)sjb::segsort_big_kernel, big_smem)) return rc;
  sjb::segsort_big_kernel<<<sjb_sm_count(current_device()), sjb::kSortBigThreads, big_smem, st>>>(
      c.rowoff, keys, d_lefts, d_rights, d_sims, c.bigrows, c.nbig, args->left_base,
      args->n_right);
  SJB_CK_LAUNCH("segsort_big");
  sjb::join_finalize_kernel<<<1, 256, 0, st>>>(c.cta, pl.grid, pl.seg_cap, c.rowoff, nl,
                                               args->out_cap, info);
  SJB_CK_LAUNCH("finalize");
  return SJB_OK;
}

}  // namespace

extern "C" {

int sjb_join_begin(const sjb_join_args* args, void* d_workspace, int64_t workspace_bytes,
                   void* stream) {
  JoinCtx c;
  if (int rc = join_ctx(args, d_workspace, workspace_bytes, &c)) return rc;
  if (c.empty) return SJB_OK;
  return join_begin(args, c, as_stream(stream));
}

int sjb_join_filter_tiles(const float* d_l32, const void* d_l16, const float* d_r32,
                          const void* d_r16, const sjb_join_args* args, void* d_workspace,
                          int64_t workspace_bytes, int64_t tile_begin, int64_t tile_end,
                          void* stream) {
  JoinCtx c;
  if (int rc = join_ctx(args, d_workspace, workspace_bytes, &c)) return rc;
  if (c.empty) return SJB_OK;
  return join_filter(d_l32, d_l16, d_r32, d_r16, args, c, tile_begin, tile_end, as_stream(stream));
}

int sjb_join_finish(const float* d_l32, const float* d_r32, const sjb_join_args* args,
                    void* d_workspace, int64_t workspace_bytes, uint64_t* d_lefts,
                    uint64_t* d_rights, float* d_sims, void* d_info, void* stream) {
  if (!d_info) return fail(SJB_E_INVALID, "null info");
  JoinCtx c;
  if (int rc = join_ctx(args, d_workspace, workspace_bytes, &c)) return rc;
  cudaStream_t st = as_stream(stream);
  int64_t* info = reinterpret_cast<int64_t*>(d_info);
  if (c.empty) {
    SJB_CK(cudaMemsetAsync(info, 0, 5 * 8, st));
    return SJB_OK;
  }
  return join_finish(d_l32, d_r32, args, c, d_lefts, d_rights, d_sims, info, st);
}

int sjb_join_prepared_async(const float* d_l32, const void* d_l16, const float* d_r32,
                            const void* d_r16, const sjb_join_args* args, void* d_workspace,
                            int64_t workspace_bytes, uint64_t* d_lefts, uint64_t* d_rights,
                            float* d_sims, void* d_info, void* stream) {
  if (!args || !d_info) return fail(SJB_E_INVALID, "null args/info");
  JoinCtx c;
  if (int rc = join_ctx(args, d_workspace, workspace_bytes, &c)) return rc;
  cudaStream_t st = as_stream(stream);
  int64_t* info = reinterpret_cast<int64_t*>(d_info);
  if (c.empty) {
    SJB_CK(cudaMemsetAsync(info, 0, 5 * 8, st));
    return SJB_OK;
  }
  if (int rc = join_begin(args, c, st)) return rc;
  if (int rc = join_filter(d_l32, d_l16, d_r32, d_r16, args, c, 0,
                           sjb::ceil_div(args->n_right, sjb::kTileRows), st))
    return rc;
  return join_finish(d_l32, d_r32, args, c, d_lefts, d_rights, d_sims, info, st);
}

int sjb_join_prepared(const float* d_l32, const void* d_l16, const float* d_r32,
                      const void* d_r16, const sjb_join_args* args, void* d_workspace,
                      int64_t workspace_bytes, uint64_t* d_lefts, uint64_t* d_rights,
                      float* d_sims, sjb_join_info* info, void* stream) {
  if (!info) return fail(SJB_E_INVALID, "null info");
  void* d_info = nullptr;
  cudaStream_t st = as_stream(stream);
  SJB_CK(cudaMallocAsync(&d_info, 64, st));
  int rc = sjb_join_prepared_async(d_l32, d_l16, d_r32, d_r16, args, d_workspace, workspace_bytes,
                                   d_lefts, d_rights, d_sims, d_info, stream);
  if (rc == SJB_OK) {
    int64_t h[5];
    SJB_CK(cudaMemcpyAsync(h, d_info, 40, cudaMemcpyDeviceToHost, st));
    SJB_CK(cudaStreamSynchronize(st));
    info->n_matches = h[0];
    info->n_candidates = h[1];
    info->cand_needed = h[2];
    info->overflow = reinterpret_cast<int32_t*>(h + 3)[0];
    info->grid = reinterpret_cast<int32_t*>(h + 3)[1];
  }
  cudaFreeAsync(d_info, st);
  return rc;
}

int sjb_tile_dot(const float* d_left, int64_t lda, const float* d_bt, int64_t ldb, int64_t nl,
                 int64_t nr, int64_t dim, float* d_out, int64_t ldo, void* stream) {
  if (nl <= 0 || nr <= 0) return SJB_OK;
  dim3 grid((unsigned)sjb::ceil_div(nr, sjb::kTD), (unsigned)sjb::ceil_div(nl, sjb::kTD));
  sjb::tile_dot_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_left, lda, d_bt, ldb, nl, nr,
                                                             (int)dim, d_out, ldo);
  SJB_CK_LAUNCH("tile_dot");
  return SJB_OK;
}

// persistent grid for vm_rows_kernel: one wave (the CTAs that fit per SM,
// from the occupancy calculator), fewer when the rows run out
static unsigned vm_grid(int64_t n, const void* kernel, int* per_sm) {
  if (*per_sm == 0) {
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, sjb::kVmWarps * 32, 0);
    *per_sm = v > 0 ? v : 1;
  }
  const int64_t groups = sjb::ceil_div(n > 0 ? n : 1, 32);
  const int64_t need = sjb::ceil_div(groups, sjb::kVmWarps);
  const int64_t cap = (int64_t)sjb_sm_count(current_device()) * *per_sm;
  return (unsigned)(need < cap ? need : cap);
}
static int vm_per_sm_cos = 0, vm_per_sm_dot = 0;

int sjb_cosine_vm(const float* d_a, const float* d_m, int64_t n, int64_t dim, float* d_out,
                  int* d_flags, void* stream) {
  if (n < 0 || dim < 1) return fail(SJB_E_INVALID, "bad shape");
  if (!d_flags) return fail(SJB_E_INVALID, "null flags");
  sjb::vm_rows_kernel<true><<<vm_grid(n, (const void*)sjb::vm_rows_kernel<true>, &vm_per_sm_cos), sjb::kVmWarps * 32, 0, as_stream(stream)>>>(
      d_a, d_m, n, (int)dim, d_out, d_flags);
  SJB_CK_LAUNCH("cosine_vm");
  return SJB_OK;
}

int sjb_dots_vm(const float* d_a, const float* d_m, int64_t n, int64_t dim, float* d_out,
                void* stream) {
  if (n <= 0) return SJB_OK;
  sjb::vm_rows_kernel<false><<<vm_grid(n, (const void*)sjb::vm_rows_kernel<false>, &vm_per_sm_dot), sjb::kVmWarps * 32, 0, as_stream(stream)>>>(
      d_a, d_m, n, (int)dim, d_out, nullptr);
  SJB_CK_LAUNCH("dots_vm");
  return SJB_OK;
}

int64_t sjb_scan_hits_workspace_bytes(int64_t nl) {
  const size_t n = (size_t)(nl > 0 ? nl : 0);
  const size_t nb = sjb::ceil_div((int64_t)n, sjb::kScanBlock) + 1;
  return (int64_t)(align256(n * 4) + align256((n + 1) * 8) + align256((nb + 1) * 8));
}

int sjb_scan_hits(const float* d_buf, int64_t nl, int64_t nr, float theta, uint64_t left0,
                  uint64_t right0, uint64_t* d_lefts, uint64_t* d_rights, float* d_sims,
                  int64_t cap, int64_t* count, void* d_workspace, int64_t workspace_bytes,
                  void* stream) {
  if (!count) return fail(SJB_E_INVALID, "null count");
  *count = 0;
  if (nl <= 0 || nr <= 0) return SJB_OK;
  if (workspace_bytes < sjb_scan_hits_workspace_bytes(nl))
    return fail(SJB_E_INVALID, "scan_hits workspace too small");
  cudaStream_t st = as_stream(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_workspace);
  const size_t n = (size_t)nl;
  uint32_t* rowcount = reinterpret_cast<uint32_t*>(ws);
  uint64_t* rowoff = reinterpret_cast<uint64_t*>(ws + align256(n * 4));
  uint64_t* bsums = reinterpret_cast<uint64_t*>(ws + align256(n * 4) + align256((n + 1) * 8));
  const unsigned blocks = (unsigned)sjb::ceil_div(nl, 8);
  sjb::dense_count_kernel<<<blocks, 256, 0, st>>>(d_buf, nl, nr, theta, rowcount);
  SJB_CK_LAUNCH("dense_count");
  if (int rc = run_scan(rowcount, nl, rowoff, nullptr, bsums, st)) return rc;
  uint64_t total = 0;
  SJB_CK(cudaMemcpyAsync(&total, rowoff + nl, 8, cudaMemcpyDeviceToHost, st));
  SJB_CK(cudaStreamSynchronize(st));
  *count = (int64_t)total;
  if (d_lefts == nullptr || (int64_t)total > cap) return SJB_OK;
  sjb::dense_fill_kernel<<<blocks, 256, 0, st>>>(d_buf, nl, nr, theta, rowoff, left0, right0,
                                                 d_lefts, d_rights, d_sims);
  SJB_CK_LAUNCH("dense_fill");
  SJB_CK(cudaStreamSynchronize(st));
  return SJB_OK;
}

// ----------------------------------------------------------- matches file
int64_t sjb_matches_csv_workspace_bytes(int64_t n) {
  const int64_t ng = sjb::ceil_div(n > 0 ? n : 0, sjb::fmt::kLines);
  const int64_t nb = sjb::ceil_div(ng, sjb::kScanBlock) + 1;
  const size_t nl = (size_t)(n > 0 ? n : 0);
  return (int64_t)(align256((size_t)ng * 4) + align256((size_t)(ng + 1) * 8) +
                   align256((size_t)(nb + 1) * 8) + align256(nl * 8) + align256(nl * 4));
}

// workspace: group lengths | group offsets | scan block sums | digits | meta
struct CsvWs {
  uint32_t* glen;
  uint64_t* goff;
  uint64_t* bsums;
  uint64_t* digs;
  uint32_t* meta;
};

static CsvWs csv_ws(const void* base, int64_t n) {
  uint8_t* ws = reinterpret_cast<uint8_t*>(const_cast<void*>(base));
  const int64_t ng = sjb::ceil_div(n, sjb::fmt::kLines);
  const int64_t nb = sjb::ceil_div(ng, sjb::kScanBlock) + 1;
  CsvWs w;
  size_t o = 0;
  w.glen = reinterpret_cast<uint32_t*>(ws + o);
  o += align256((size_t)ng * 4);
  w.goff = reinterpret_cast<uint64_t*>(ws + o);
  o += align256((size_t)(ng + 1) * 8);
  w.bsums = reinterpret_cast<uint64_t*>(ws + o);
  o += align256((size_t)(nb + 1) * 8);
  w.digs = reinterpret_cast<uint64_t*>(ws + o);
  o += align256((size_t)n * 8);
  w.meta = reinterpret_cast<uint32_t*>(ws + o);
  return w;
}

static int csv_check(const uint64_t* l, const uint64_t* r, const float* s, int64_t n,
                     int64_t workspace_bytes) {
  if (n < 0) return fail(SJB_E_INVALID, "negative match count");
  if (n > 0 && (!l || !r || !s)) return fail(SJB_E_INVALID, "null match column");
  if (workspace_bytes < sjb_matches_csv_workspace_bytes(n))
    return fail(SJB_E_INVALID, "matches_csv workspace too small");
  if (sjb::ceil_div(n, sjb::fmt::kLines) > (int64_t)sjb::kScanBlock * sjb::kScanBlock)
    return fail(SJB_E_UNSUPPORTED, "too many matches for one call");
  return SJB_OK;
}

int sjb_matches_csv_layout(const uint64_t* d_lefts, const uint64_t* d_rights,
                           const float* d_sims, int64_t n, void* d_workspace,
                           int64_t workspace_bytes, int64_t* out_bytes, void* stream) {
  if (!out_bytes) return fail(SJB_E_INVALID, "null out_bytes");
  *out_bytes = 0;
  if (int rc = csv_check(d_lefts, d_rights, d_sims, n, workspace_bytes)) return rc;
  if (n == 0) return SJB_OK;
  cudaStream_t st = as_stream(stream);
  const int64_t ng = sjb::ceil_div(n, sjb::fmt::kLines);
  const CsvWs w = csv_ws(d_workspace, n);
  sjb::fmt::csv_layout_kernel<<<(unsigned)ng, sjb::fmt::kLines, 0, st>>>(
      d_lefts, d_rights, d_sims, n, w.glen, w.digs, w.meta);
  SJB_CK_LAUNCH("csv_layout");
  if (int rc = run_scan(w.glen, ng, w.goff, nullptr, w.bsums, st)) return rc;
  uint64_t total = 0;
  SJB_CK(cudaMemcpyAsync(&total, w.goff + ng, 8, cudaMemcpyDeviceToHost, st));
  SJB_CK(cudaStreamSynchronize(st));
  *out_bytes = (int64_t)total;
  return SJB_OK;
}

int sjb_matches_csv_write(const uint64_t* d_lefts, const uint64_t* d_rights,
                          const float* d_sims, int64_t n, const void* d_workspace,
                          int64_t workspace_bytes, uint8_t* d_out, int64_t out_cap,
                          void* stream) {
  if (int rc = csv_check(d_lefts, d_rights, d_sims, n, workspace_bytes)) return rc;
  if (n == 0) return SJB_OK;
  if (!d_out) return fail(SJB_E_INVALID, "null output buffer");
  cudaStream_t st = as_stream(stream);
  const int64_t ng = sjb::ceil_div(n, sjb::fmt::kLines);
  const CsvWs w = csv_ws(d_workspace, n);
  uint64_t total = 0;  // checked against the capacity: a layout from other inputs is an error
  SJB_CK(cudaMemcpyAsync(&total, w.goff + ng, 8, cudaMemcpyDeviceToHost, st));
  SJB_CK(cudaStreamSynchronize(st));
  if ((int64_t)total > out_cap) return fail(SJB_E_INVALID, "output buffer too small");
  sjb::fmt::csv_write_kernel<<<(unsigned)ng, sjb::fmt::kLines, 0, st>>>(
      d_lefts, d_rights, w.digs, w.meta, n, w.goff, d_out);
  SJB_CK_LAUNCH("csv_write");
  return SJB_OK;
}

}  // extern "C"
