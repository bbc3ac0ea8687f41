// sjb_join3.cu -- threshold filter + canonical recheck for wide embeddings
// (kpad > 128, e.g. BASELINE cfg4 d = 768), K-streaming.
//
// Filter.  The resident-R design of sjb_join.cu needs the whole 256 x kpad R
// block in shared memory (384 KB at d = 768), so here both operands stream
// through the ring in K chunks of 64 elements: a stage = the R block's chunk
// (256 rows x 64, 32 KB) + the S tile's chunk (256 rows x 64, 32 KB), both
// contiguous in the [k-group][256][8] operand image.  Per chunk, 2 x 4
// UMMA_128x256x16 (one per R half) accumulate into the two 256-column halves
// of TMEM; the output tile is 256 x 256 and K/64 chunks long (12 at d = 768:
// ~12k MMA cycles), so one accumulator stage suffices: each TMEM half is
// handed back (acc_empty[h]) as soon as the epilogue has drained it, so the
// next tile's first MMAs overlap the emission of the previous one.  The
// epilogue and the candidate segments are those of sjb_join.cu.
//
// Recheck.  At d = 768 a candidate's canonical chain reads 2 x 3 KB of fp32
// rows, and clustered data gives ~600 candidates per 256 x 256 tile, so
// per-candidate gathers from L2 (the fused recheck of sjb_join.cu) cost
// ~6 KB/candidate of L2 traffic -- 5x the filter's own.  The default here
// is therefore a second kernel, `recheck_kernel`: the filter records where
// each tile's candidates start in its segment (`tile_off`), and the recheck
// walks the same tiles, stages the tile's fp32 R and S rows in 32-element K
// chunks through shared memory (double-buffered cp.async) and advances every
// candidate's sequential FMA chain chunk by chunk -- the same d = 0..dim-1
// order, so the value is bitwise `sj_dot_seq` (_kernelcore.c:101-106).  L2
// traffic drops to ~1.5 MB per tile (~2.5 KB per candidate).  Tiles with few
// candidates skip the staging and gather directly.  The fused variant
// (kFused = true, 10 recheck warps) is kept for A/B measurement.
#include "sjb_common.cuh"

namespace sjb {
namespace wide {

#ifndef SJB_WIDE_EPI
#define SJB_WIDE_EPI 8
#endif
constexpr int kEpiWarps = SJB_WIDE_EPI;
static_assert(kEpiWarps == 8 || kEpiWarps == 16, "SJB_WIDE_EPI: 8 or 16");
// 8 warps drain 64-column chunks, 16 warps 32-column chunks (half the live
// accumulator registers); either way a warp has two chunks per TMEM half
constexpr int kCW = kEpiWarps == 8 ? 64 : 32;
constexpr int kChunksPerWarp = 2;
// first column (within a half) of chunk k of the warps of column group cq0
__device__ __forceinline__ int chunk_col(int cq0, int k) {
  return kEpiWarps == 8 ? (cq0 + 2 * k) * 64 : cq0 * 64 + k * 32;
}
template <bool kFused>
struct Cfg {
  static constexpr int kRecheckWarps = kFused ? 10 : 0;
  static constexpr int kThreads = 32 * (2 + kEpiWarps + kRecheckWarps);
};
#ifndef SJB_WIDE_KCHUNK
#define SJB_WIDE_KCHUNK 64
#endif
constexpr int kKChunk = SJB_WIDE_KCHUNK;              // K elements per stage
constexpr int kMaxStages = 6 * 64 / kKChunk;          // ring depth cap (same bytes)
constexpr int kChunkBytes = kTileRows * kKChunk * 2;  // 32 KB per operand

struct Params {
  const op16_t* a16;
  const op16_t* b16;
  int64_t n_a, n_b;
  int kpad;              // multiple of 64
  int n_ablk, n_btiles;  // 256-row blocks / tiles
  int tiles_per_chunk;
  int tile_begin;        // first S tile of this launch
  int append;            // 1: continue the segments of an earlier launch
  int64_t n_items;
  int stages;
  float cutoff;
  const float* row_err;   // per-row band (or nullptr: uniform cutoff)
  const float* tile_err;
  float slack;
  uint64_t* cand;
  uint64_t seg_cap;
  unsigned long long* cta_count;
  uint32_t* tile_off;    // [grid][tile_stride]: segment offset at each tile start (+ end)
  int64_t tile_stride;
  const float* l32;
  const float* r32;
  int dim;
  float theta;
  uint32_t* sims_bits;
  uint32_t* rowcount;
  int debug;  // diagnostics, results invalid: 1 fused recheck warps idle / no emission,
             // 2 no TMEM drain, 20 no operand traffic after the ring filled once
  // raw-operand mode (bf16 inputs, sjb_prepare_bf16): the operands are the
  // raw bf16 rows and the epilogue normalises after the GEMM,
  // approx = (acc * inv_a[i]) * inv_b[j]; nullptr: normalised operands
  const float* inv_a;
  const float* inv_b;
  // tolerance emission (sims_mode 1, raw mode): pairs with approx >= hi_cut
  // are final (sim = approx, counted here); pairs in [cutoff, hi_cut) are
  // pending -- their slots go to the CTA's pending list for the canonical
  // recheck (recheck_pending_kernel)
  int tol;
  float hi_cut;
  uint32_t* pend;        // [grid][seg_cap] pending slot indices
  uint32_t* pend_count;  // [grid] pending entries of this launch
};

// Tolerance emission: each epilogue lane's 32-column scratch row (pitch 33
// floats: a lane's row is conflict-free against the other lanes')
constexpr int kTolPitch = 33;
constexpr uint32_t kTolScratchBytes = kEpiWarps * 32 * kTolPitch * 4;

// Without the tolerance scratch the same place holds each epilogue warp's copy
// of the tile's inverse norms (raw-operand mode, canonical sims): its chunks'
// 64 floats each, prefetched before the accumulator wait and read as
// shared-memory broadcasts -- the per-chunk __ldg's of inv_b sat on the tile's
// critical path (one L2 round trip per chunk before the half is released).
constexpr uint32_t kInvStageBytes = kEpiWarps * 32 * 16;

__host__ __device__ inline uint32_t smem_bytes(int stages, bool tol = false) {
  return (uint32_t)stages * 2 * kChunkBytes + (4 + 2 * stages) * 8 + 32 +
         (tol ? kTolScratchBytes : kInvStageBytes);
}

// Max tiles one CTA walks in one launch (+1 for the end offset), for any
// S-tile range of the join and chunking <= max_tpc: a launch over `range`
// tiles with chunk tpc has n_ablk * ceil(range / tpc) items, so a CTA walks
// <= ceil(items / grid) * tpc <= n_ablk * (range + tpc) / grid + tpc tiles.
__host__ __device__ inline int64_t tile_stride(int64_t n_ablk, int64_t n_btiles, int grid,
                                               int max_tpc) {
  return (n_ablk * (n_btiles + max_tpc) + grid - 1) / grid + max_tpc + 1;
}

__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
}

// ---- CTA pairs (kPair): two CTAs of a cluster take R blocks 2p and 2p + 1
// against the same S tiles; each loads its own R chunk, rank 0 multicasts
// the S chunk into both CTAs' rings (the per-tile L2 operand traffic falls
// from 2 x 256 rows to 1.5 x 256 rows per CTA: the filter at d = 768 is L2
// bound).  A ring slot is refilled only when BOTH CTAs' MMAs are done with
// it: the MMA commit arrives on the slot's `empty` barrier in both CTAs
// (count 2).
__device__ __forceinline__ uint32_t cta_rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void bulk_g2s_mc(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                            uint64_t* bar, uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1], %2, [%3], %4, %5;" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "h"(mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc_elect(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}" ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

template <bool kFused, bool kPair = false>
__global__ void __launch_bounds__(Cfg<kFused>::kThreads, 1) filter_kernel(const Params p) {
  constexpr int kRecheckWarps = Cfg<kFused>::kRecheckWarps;
  static_assert(!(kFused && kPair), "pairs: separate recheck only");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;  // stage s: A chunk at s*64K, B chunk at s*64K + 32K
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * 2 * kChunkBytes);
  uint64_t* acc_full = bars + 0;
  uint64_t* acc_empty = bars + 1;  // [2]: one per TMEM half
  uint64_t* full = bars + 4;
  uint64_t* empty = bars + 4 + p.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 + 2 * p.stages);
  uint32_t* cta_cnt = tmem_slot + 2;
  uint32_t* cta_sat = tmem_slot + 3;
  uint32_t* epi_done = tmem_slot + 4;
  uint32_t* pend_cnt = tmem_slot + 5;
  float* tol_scratch = reinterpret_cast<float*>(tmem_slot + 8);   // kTolScratchBytes (tol only)
  float4* inv_stage = reinterpret_cast<float4*>(tmem_slot + 8);   // kInvStageBytes (!tol, raw mode)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(acc_full, 1);
    mbar_init(&acc_empty[0], kEpiWarps);
    mbar_init(&acc_empty[1], kEpiWarps);
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPair ? 2 : 1);
    }
    init_segment_count(p.cta_count, p.append != 0, cta_cnt, cta_sat);
    *epi_done = 0u;
    *pend_cnt = 0u;
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_barrier();   // the peer's barriers exist before any multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // work items: (R block, S chunk), S-chunk-major.  kPair: the pair's items
  // are (R block pair, S chunk); this CTA takes block 2 bp + rank (a block
  // past the end -- odd block count -- is a phantom: loaded, never emitted)
  const uint32_t rank = kPair ? cta_rank_in_cluster() : 0u;
  const int nb = kPair ? (p.n_ablk + 1) / 2 : p.n_ablk;
  const int64_t n_items = kPair ? (int64_t)nb * (p.n_items / p.n_ablk) : p.n_items;
  const int64_t item0 = kPair ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
  const int64_t item_step = kPair ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;
  auto item_rb = [&](int64_t item) -> int64_t {
    return kPair ? 2 * (item % nb) + rank : item % nb;
  };
  const int nchunks = p.kpad / kKChunk;
  const size_t tile_elems = (size_t)kTileRows * p.kpad;
  const size_t chunk_elems = (size_t)kChunkBytes / 2;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer
      const uint64_t pol_a = policy_evict_last();
      const uint64_t pol_b = policy_evict_normal();
      int s = 0;
      uint32_t ph = 0;
      int64_t fills = 0;
      for (int64_t item = item0; item < n_items; item += item_step) {
        const int64_t rb = mn<int64_t>(item_rb(item), p.n_ablk - 1), sc = item / nb;
        const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
        for (int64_t t = t0; t < t1; t++) {
          for (int c = 0; c < nchunks; c++, fills++) {
            mbar_wait(&empty[s], ph ^ 1u);
            if (p.debug == 20 && fills >= p.stages) {   // diagnostics: no operand traffic
              mbar_arrive(&full[s]);                     // after the ring filled once
              if (++s == p.stages) {
                s = 0;
                ph ^= 1u;
              }
              continue;
            }
            mbar_arrive_expect_tx(&full[s], 2 * kChunkBytes);
            uint8_t* dst = ring + (size_t)s * 2 * kChunkBytes;
            bulk_g2s(dst, p.a16 + rb * tile_elems + c * chunk_elems, kChunkBytes, &full[s], pol_a);
            if (!kPair)
              bulk_g2s(dst + kChunkBytes, p.b16 + t * tile_elems + c * chunk_elems, kChunkBytes,
                       &full[s], pol_b);
            else if (rank == 0)   // the S chunk into both CTAs' slot s
              bulk_g2s_mc(dst + kChunkBytes, p.b16 + t * tile_elems + c * chunk_elems, kChunkBytes,
                          &full[s], (uint16_t)0x3, pol_b);
            if (++s == p.stages) {
              s = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    // whole warp, warp-uniform; one elected lane issues (lean issue)
    const uint32_t idesc = umma_idesc_f16_f32(128, 256, p.inv_a != nullptr);
    const uint32_t lbo = kTileRows * 16, sbo = 128;
    const uint64_t kstep = (2 * lbo) >> 4, half_step = (128 * 16) >> 4;
    const uint64_t ring_desc = umma_desc_kmajor_noswz(smem_u32(ring), lbo, sbo);
    const uint64_t stage_step = (2 * kChunkBytes) >> 4, b_off = kChunkBytes >> 4;
    int s = 0;
    uint32_t ph = 0, tile_it = 0;
    for (int64_t item = item0; item < n_items; item += item_step) {
      const int64_t sc = item / nb;
      const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
      const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
      for (int64_t t = t0; t < t1; t++, tile_it++) {
        for (int c = 0; c < nchunks; c++) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = ring_desc + (uint64_t)s * stage_step, bd = ad + b_off;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            if (c == 0) {  // half h of TMEM drained by the epilogue?
              mbar_wait(&acc_empty[h], (tile_it & 1u) ^ 1u);
              tc_fence_after();
            }
#pragma unroll
            for (int kk = 0; kk < kKChunk / 16; kk++)
              tc_mma_f16_elect(tmem_base + h * 256, ad + h * half_step + kk * kstep,
                                bd + kk * kstep, idesc, (c | kk) ? 1u : 0u);
          }
          if (kPair)
            tc_commit_mc_elect(&empty[s], (uint16_t)0x3);   // both CTAs' slot s
          else
            tc_commit_elect(&empty[s]);
          if (++s == p.stages) {
            s = 0;
            ph ^= 1u;
          }
        }
        tc_commit_elect(acc_full);
      }
    }
  } else if (warp >= 2 + kEpiWarps) {
    // ------------------------------------------- fused recheck (kFused only)
    const uint64_t seg_cap = p.seg_cap;
    if (p.debug != 1)
      recheck_loop(p.cand + (uint64_t)blockIdx.x * seg_cap,
                   p.sims_bits + (uint64_t)blockIdx.x * seg_cap, seg_cap, cta_cnt, epi_done,
                   (uint32_t)kEpiWarps, warp - 2 - kEpiWarps, kRecheckWarps, p.l32, p.r32, p.dim,
                   p.theta, p.rowcount, p.append ? (uint64_t)p.cta_count[blockIdx.x] : 0ull);
  } else {
    // ---------------------------------------------------------- epilogue
    // warp (q, c): TMEM lanes 32q..32q+31 x column chunks c, c + 2 (64 each)
    // of BOTH halves; a half is handed back after its last chunk is loaded
    const int ew = warp - 2;
    const int cq0 = ew >> 2, q = warp & 3;
    const uint32_t lane_base = (uint32_t)q * 32;
    uint64_t* seg = p.cand + (uint64_t)blockIdx.x * p.seg_cap;
    const uint64_t seg_cap = p.seg_cap;
    uint32_t* toff = kFused ? nullptr : p.tile_off + (int64_t)blockIdx.x * p.tile_stride;
    uint32_t tile_it = 0;
    for (int64_t item = item0; item < n_items; item += item_step) {
      const int64_t rb = item_rb(item), sc = item / nb;   // rb >= n_ablk: phantom (no rows)
      const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
      const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
      uint32_t fin0 = 0u, fin1 = 0u;   // tolerance emission: this lane's rows' final matches
      for (int64_t t = t0; t < t1; t++, tile_it++) {
        const bool stage_inv = p.inv_a != nullptr && !p.tol;
        float4 inv4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (stage_inv && lane < 2 * (kCW / 4))   // lands during the accumulator wait
          inv4 = __ldg(reinterpret_cast<const float4*>(
                           p.inv_b + t * kTileRows + chunk_col(cq0, lane / (kCW / 4))) +
                       (lane % (kCW / 4)));
        mbar_wait(acc_full, tile_it & 1u);
        tc_fence_after();
        if (stage_inv) {
          __syncwarp();   // the previous tile's reads are done
          inv_stage[ew * 32 + lane] = inv4;
          __syncwarp();
        }
        if (!kFused) {
          // every epilogue warp is done with the previous tile's emission:
          // the counter is this tile's first slot
          epi_bar();
          if (ew == 0 && lane == 0) toff[tile_it] = *(volatile uint32_t*)cta_cnt;
        }
#pragma unroll 1
        for (int h = 0; h < 2; h++) {
          const int64_t gi64 = rb * kTileRows + h * 128 + lane_base + lane;
          const float cutoff =
              row_cutoff(p.cutoff, p.theta, p.slack, p.row_err, p.tile_err, gi64, p.n_a, t);
          const float inv_i = (p.inv_a != nullptr && gi64 < p.n_a) ? __ldg(p.inv_a + gi64) : 1.0f;
#pragma unroll 1
          for (int k = 0; k < kChunksPerWarp; k++) {
            const int cc = chunk_col(cq0, k);
            const uint32_t taddr = tmem_base + (lane_base << 16) + h * 256 + cc;
            if (p.debug == 2) {   // diagnostics: no drain (MMA + operand delivery only)
              if (k == kChunksPerWarp - 1) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_relaxed(&acc_empty[h]);
              }
              continue;
            }
            float v[kCW];
            SJB_TMEM_LD32(taddr, v, 0);
            if (kCW == 64) SJB_TMEM_LD32(taddr + 32, v, kCW - 32);
            tc_wait_ld();
            if (k == kChunksPerWarp - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_relaxed(&acc_empty[h]);
            }
            if (p.debug == 1) {   // diagnostics: drain, no emission (results invalid)
              float m = v[0];
#pragma unroll
              for (int e = 1; e < kCW; e++) m = fmaxf(m, v[e]);
              if (m > 3.0e38f) cta_sat[0] = 1u;   // never true: keeps the loads live
              continue;
            }
            const int64_t col_lim = p.n_b - t * kTileRows - cc;
            if (p.inv_a != nullptr) {
              // normalise after the GEMM: (acc * inv_i) * inv_j (inv_b is
              // padded to whole tiles, zero past n_b)
              const float4* ib = reinterpret_cast<const float4*>(p.inv_b + t * kTileRows + cc);
              const float4* is = inv_stage + ew * 32 + (kCW / 4) * k;
#pragma unroll
              for (int q4 = 0; q4 < kCW / 4; q4++) {
                const float4 w = stage_inv ? is[q4] : __ldg(ib + q4);
                v[4 * q4 + 0] = __fmul_rn(__fmul_rn(v[4 * q4 + 0], inv_i), w.x);
                v[4 * q4 + 1] = __fmul_rn(__fmul_rn(v[4 * q4 + 1], inv_i), w.y);
                v[4 * q4 + 2] = __fmul_rn(__fmul_rn(v[4 * q4 + 2], inv_i), w.z);
                v[4 * q4 + 3] = __fmul_rn(__fmul_rn(v[4 * q4 + 3], inv_i), w.w);
              }
            }
            if (p.tol) {
              const uint32_t f = emit_row_chunk_tol<kCW>(v, gi64 < p.n_a, cutoff, p.hi_cut, (uint32_t)gi64,
                                             (uint32_t)(t * kTileRows + cc), col_lim,
                                             cta_cnt, cta_sat, seg, seg_cap,
                                             p.sims_bits + (uint64_t)blockIdx.x * seg_cap,
                                             pend_cnt, p.pend + (uint64_t)blockIdx.x * seg_cap,
                                             tol_scratch + (ew * 32 + lane) * kTolPitch);
              if (h) fin1 += f; else fin0 += f;
            } else
              emit_row_chunk<kCW>(v, gi64 < p.n_a, cutoff, (uint32_t)gi64,
                                  (uint32_t)(t * kTileRows + cc), col_lim, cta_cnt, cta_sat,
                                  seg, seg_cap);
          }
        }
      }
      if (p.tol) {   // rows >= n_a (phantom blocks included) never have finals
        if (fin0) atomicAdd(p.rowcount + rb * kTileRows + lane_base + lane, fin0);
        if (fin1) atomicAdd(p.rowcount + rb * kTileRows + 128 + lane_base + lane, fin1);
      }
    }
    if (!kFused) {
      epi_bar();
      if (ew == 0 && lane == 0) toff[tile_it] = *(volatile uint32_t*)cta_cnt;
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      atomicAdd(epi_done, 1u);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
  if (threadIdx.x == 0) {
    p.cta_count[blockIdx.x] = *cta_sat ? ~0ull >> 1 : (unsigned long long)*cta_cnt;
    if (p.tol) p.pend_count[blockIdx.x] = *pend_cnt;
  }
  if (kPair) cluster_barrier();   // no peer multicast or commit targets an exited CTA
}

// ------------------------------------------------------------- recheck
constexpr int kRcThreads = 512;
constexpr int kRcKC = 32;             // K elements per staged chunk
constexpr int kRcPitch = kRcKC + 4;   // floats per staged row (16 B aligned, bank spread)
constexpr int kRcCpt = 4;             // candidates per thread per pass
constexpr int kRcPass = kRcThreads * kRcCpt;
constexpr int kRcDirect = 128;        // fewer candidates than this: gather, no staging
constexpr int kRcBufFloats = 2 * kTileRows * kRcPitch;  // A + B rows of one chunk

__host__ __device__ constexpr uint32_t recheck_smem_bytes() {
  return 2u * kRcBufFloats * 4u;
}

struct RecheckParams {
  const uint64_t* cand;
  uint64_t seg_cap;
  const unsigned long long* cta_count;
  const uint32_t* tile_off;
  int64_t tile_stride;
  int64_t n_items;
  int n_ablk, n_btiles, tiles_per_chunk, tile_begin;
  int64_t n_a, n_b;
  const float* l32;
  const float* r32;
  int dim;
  float theta;
  uint32_t* sims_bits;
  uint32_t* rowcount;
  uint32_t direct_max;  // tiles with fewer candidates gather instead of staging
  unsigned int* work;   // recheck_group_kernel: dynamic item counter (zeroed per launch)
  int filter_grid;      // the filter's grid (item -> owning segment)
};

__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Stage K chunk `ch` of the tile's R rows (r0.., nr_a valid) and S rows.
__device__ __forceinline__ void stage_chunk(float* buf, const float* l32, const float* r32,
                                            int64_t r0, int nr_a, int64_t c0, int nr_b, int dim,
                                            int ch, bool vec) {
  const int k0 = ch * kRcKC;
  const int kc = mn(kRcKC, dim - k0);
  float* as = buf;
  float* bs = buf + kTileRows * kRcPitch;
  if (vec) {  // dim % 4 == 0: rows and chunk starts are 16 B aligned
    const int q4 = kc >> 2;
    for (int idx = threadIdx.x; idx < 2 * kTileRows * 8; idx += kRcThreads) {
      const int side = idx >= kTileRows * 8;
      const int e = side ? idx - kTileRows * 8 : idx;
      const int r = e >> 3, q = e & 7;
      if (q >= q4) continue;
      if (!side) {
        if (r < nr_a) cp_async16(as + r * kRcPitch + 4 * q, l32 + (r0 + r) * dim + k0 + 4 * q);
      } else {
        if (r < nr_b) cp_async16(bs + r * kRcPitch + 4 * q, r32 + (c0 + r) * dim + k0 + 4 * q);
      }
    }
  } else {
    for (int idx = threadIdx.x; idx < 2 * kTileRows * kRcKC; idx += kRcThreads) {
      const int side = idx >= kTileRows * kRcKC;
      const int e = side ? idx - kTileRows * kRcKC : idx;
      const int r = e / kRcKC, q = e % kRcKC;
      if (q >= kc) continue;
      if (!side) {
        if (r < nr_a) cp_async4(as + r * kRcPitch + q, l32 + (r0 + r) * dim + k0 + q);
      } else {
        if (r < nr_b) cp_async4(bs + r * kRcPitch + q, r32 + (c0 + r) * dim + k0 + q);
      }
    }
  }
  cp_async_commit();
}

__device__ __forceinline__ void finish_candidate(uint32_t* sims, uint64_t slot, uint32_t gi,
                                                 float x, float theta, uint32_t* rowcount) {
  const bool ok = x >= theta;
  sims[slot] = ok ? __float_as_uint(x) : kRejected;
  if (ok) atomicAdd(rowcount + gi, 1u);
}

// One CTA per filter segment; walks the segment's tiles in the filter's order.
// cp.async staging, any dim (the TMA kernel below needs dim % 4 == 0).
__global__ void __launch_bounds__(kRcThreads, 1) recheck_generic_kernel(const RecheckParams p) {
  extern __shared__ __align__(16) float rsm[];
  const int c = blockIdx.x;
  const unsigned long long cc = p.cta_count[c];
  if (cc > p.seg_cap) return;  // saturated segment: the join is retried with room
  const uint64_t* seg = p.cand + (uint64_t)c * p.seg_cap;
  uint32_t* sims = p.sims_bits + (uint64_t)c * p.seg_cap;
  const uint32_t* toff = p.tile_off + (int64_t)c * p.tile_stride;
  const int dim = p.dim;
  const float theta = p.theta;
  const int nch = (dim + kRcKC - 1) / kRcKC;
  const bool vec = (dim & 3) == 0;
  const int nb = p.n_ablk;
  int64_t k = 0;
  for (int64_t item = c; item < p.n_items; item += gridDim.x) {
    const int64_t rb = item % nb, sc = item / nb;
    const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
    const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
    for (int64_t t = t0; t < t1; t++, k++) {
      const uint32_t lo = toff[k], hi = toff[k + 1];
      if (hi <= lo) continue;
      const uint32_t n = hi - lo;
      if (n < p.direct_max) {
        // ------------------------------------------------ direct gathers
        for (uint32_t s = lo + threadIdx.x; s < hi; s += kRcThreads) {
          const uint64_t u = seg[s];
          const uint32_t gi = (uint32_t)(u >> 32), gj = (uint32_t)u;
          const float x = dot_seq_dev(p.l32 + (size_t)gi * dim, p.r32 + (size_t)gj * dim, dim);
          finish_candidate(sims, s, gi, x, theta, p.rowcount);
        }
        continue;
      }
      // -------------------------------------------------- staged chunks
      const int64_t r0 = rb * kTileRows, c0 = t * kTileRows;
      const int nr_a = (int)mn<int64_t>(kTileRows, p.n_a - r0);
      const int nr_b = (int)mn<int64_t>(kTileRows, p.n_b - c0);
      for (uint32_t base = lo; base < hi; base += kRcPass) {
        uint32_t ia[kRcCpt], jb[kRcCpt];
        float acc[kRcCpt];
#pragma unroll
        for (int m = 0; m < kRcCpt; m++) {
          const uint32_t s = base + threadIdx.x + m * kRcThreads;
          acc[m] = 0.0f;
          ia[m] = jb[m] = 0xFFFFFFFFu;
          if (s < hi) {
            const uint64_t u = seg[s];
            ia[m] = (uint32_t)((u >> 32) - (uint64_t)r0) * kRcPitch;
            jb[m] = ((uint32_t)u - (uint32_t)c0) * kRcPitch;
          }
        }
        stage_chunk(rsm, p.l32, p.r32, r0, nr_a, c0, nr_b, dim, 0, vec);
        for (int ch = 0; ch < nch; ch++) {
          if (ch + 1 < nch) {
            stage_chunk(rsm + ((ch + 1) & 1) * kRcBufFloats, p.l32, p.r32, r0, nr_a, c0, nr_b,
                        dim, ch + 1, vec);
            cp_async_wait<1>();
          } else {
            cp_async_wait<0>();
          }
          __syncthreads();
          const float* as = rsm + (ch & 1) * kRcBufFloats;
          const float* bs = as + kTileRows * kRcPitch;
          const int kc = mn(kRcKC, dim - ch * kRcKC);
          if (kc == kRcKC) {
#pragma unroll
            for (int m = 0; m < kRcCpt; m++) {
              if (ia[m] == 0xFFFFFFFFu) continue;
              const float4* a4 = reinterpret_cast<const float4*>(as + ia[m]);
              const float4* b4 = reinterpret_cast<const float4*>(bs + jb[m]);
              float x = acc[m];
#pragma unroll
              for (int q = 0; q < kRcKC / 4; q++) {
                const float4 a = a4[q], b = b4[q];
                x = __fmaf_rn(a.x, b.x, x);
                x = __fmaf_rn(a.y, b.y, x);
                x = __fmaf_rn(a.z, b.z, x);
                x = __fmaf_rn(a.w, b.w, x);
              }
              acc[m] = x;
            }
          } else {
#pragma unroll
            for (int m = 0; m < kRcCpt; m++) {
              if (ia[m] == 0xFFFFFFFFu) continue;
              float x = acc[m];
              for (int q = 0; q < kc; q++) x = __fmaf_rn(as[ia[m] + q], bs[jb[m] + q], x);
              acc[m] = x;
            }
          }
          __syncthreads();  // buffer (ch & 1) is restaged at ch + 2
        }
#pragma unroll
        for (int m = 0; m < kRcCpt; m++) {
          const uint32_t s = base + threadIdx.x + m * kRcThreads;
          if (s < hi)
            finish_candidate(sims, s, (uint32_t)(r0 + ia[m] / kRcPitch), acc[m], theta,
                             p.rowcount);
        }
      }
    }
  }
}

// ------------------------------------------------ recheck, TMA-staged
// Warp 0 lane 0 streams each staged tile's fp32 R and S rows, K chunk by K
// chunk (2-D tensor TMA, box 32 x 256, 128 B swizzle: 16 B group q of row r
// lands at q ^ (r & 7), so 8 lanes reading 8 rows hit 8 bank groups when the
// rows differ mod 8), through a 3-stage mbarrier ring.  11 compute warps own
// up to 4 candidates per thread per pass and advance two chains at a time.
constexpr int kRtComputeWarps = 11;  // + producer = 384 threads (168-register cap)
constexpr int kRtThreads = 32 * (1 + kRtComputeWarps);
constexpr int kRtStages = 3;
constexpr int kRtCpt = 4;
constexpr int kRtPass = kRtComputeWarps * 32 * kRtCpt;
constexpr int kRtOpBytes = kTileRows * kRcKC * 4;  // 32 KB: 256 rows x 128 B

__host__ __device__ constexpr uint32_t recheck_tma_smem_bytes() {
  return kRtStages * 2 * kRtOpBytes + 1024 + 2 * kRtStages * 8;
}

struct RecheckTmaParams {
  RecheckParams b;
  CUtensorMap tmap_l, tmap_r;  // fp32 rows: dims {dim, n}, box {32, 256}, SWIZZLE_128B
};

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds1(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
// byte offset of element (row r, k) in a swizzled [256][32] fp32 stage
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t k) {
  return r * 128u + ((((k >> 2) ^ (r & 7u))) << 4) + (k & 3u) * 4u;
}

__global__ void __launch_bounds__(kRtThreads, 1)
    recheck_tma_kernel(const __grid_constant__ RecheckTmaParams tp) {
  const RecheckParams& p = tp.b;
  extern __shared__ uint8_t rt_raw[];
  const uint32_t raw = smem_u32(rt_raw);
  uint8_t* base = rt_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kRtStages * 2 * kRtOpBytes);
  uint64_t* empty = full + kRtStages;
  const int c = blockIdx.x;
  if (p.cta_count[c] > p.seg_cap) return;  // saturated segment: the join is retried
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRtStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kRtComputeWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t* seg = p.cand + (uint64_t)c * p.seg_cap;
  uint32_t* sims = p.sims_bits + (uint64_t)c * p.seg_cap;
  const uint32_t* toff = p.tile_off + (int64_t)c * p.tile_stride;
  const int dim = p.dim;
  const int nch = (dim + kRcKC - 1) / kRcKC;
  const int nb = p.n_ablk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int s = 0;
  uint32_t ph = 0;

  if (warp == 0) {
    if (lane != 0) return;
    // -------------------------------------------------------- producer
    int64_t k = 0;
    for (int64_t item = c; item < p.n_items; item += gridDim.x) {
      const int64_t rb = item % nb, sc = item / nb;
      const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
      const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
      for (int64_t t = t0; t < t1; t++, k++) {
        const uint32_t lo = toff[k], hi = toff[k + 1];
        if (hi <= lo || hi - lo < p.direct_max) continue;
        for (uint32_t pb = lo; pb < hi; pb += kRtPass) {
          for (int ch = 0; ch < nch; ch++) {
            mbar_wait(&empty[s], ph ^ 1u);
            mbar_arrive_expect_tx(&full[s], 2 * kRtOpBytes);
            uint8_t* dst = base + (size_t)s * 2 * kRtOpBytes;
            tma2d(dst, &tp.tmap_l, ch * kRcKC, (int)(rb * kTileRows), &full[s]);
            tma2d(dst + kRtOpBytes, &tp.tmap_r, ch * kRcKC, (int)(t * kTileRows), &full[s]);
            if (++s == kRtStages) {
              s = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------ compute
  const int ct = threadIdx.x - 32;
  constexpr int kCT = kRtComputeWarps * 32;
  const float theta = p.theta;
  int64_t k = 0;
  for (int64_t item = c; item < p.n_items; item += gridDim.x) {
    const int64_t rb = item % nb, sc = item / nb;
    const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
    const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
    for (int64_t t = t0; t < t1; t++, k++) {
      const uint32_t lo = toff[k], hi = toff[k + 1];
      if (hi <= lo) continue;
      if (hi - lo < p.direct_max) {
        for (uint32_t q = lo + ct; q < hi; q += kCT) {
          const uint64_t u = seg[q];
          const uint32_t gi = (uint32_t)(u >> 32), gj = (uint32_t)u;
          const float x = dot_seq_dev(p.l32 + (size_t)gi * dim, p.r32 + (size_t)gj * dim, dim);
          finish_candidate(sims, q, gi, x, theta, p.rowcount);
        }
        continue;
      }
      const uint32_t r0 = (uint32_t)(rb * kTileRows), c0 = (uint32_t)(t * kTileRows);
      for (uint32_t pb = lo; pb < hi; pb += kRtPass) {
        uint32_t ra[kRtCpt], rbv[kRtCpt];
        float acc[kRtCpt];
        int nm = 0;  // this thread's candidates in the pass (prefix of m)
#pragma unroll
        for (int m = 0; m < kRtCpt; m++) {
          const uint32_t q = pb + ct + m * kCT;
          acc[m] = 0.0f;
          ra[m] = rbv[m] = 0;
          if (q < hi) {
            const uint64_t u = seg[q];
            ra[m] = (uint32_t)(u >> 32) - r0;
            rbv[m] = (uint32_t)u - c0;
            nm = m + 1;
          }
        }
        for (int ch = 0; ch < nch; ch++) {
          mbar_wait(&full[s], ph);
          const uint32_t sa = smem_u32(base + (size_t)s * 2 * kRtOpBytes);
          const uint32_t sb = sa + kRtOpBytes;
          const int kc = mn(kRcKC, dim - ch * kRcKC);
          if (kc == kRcKC) {
#pragma unroll
            for (int m = 0; m < kRtCpt; m += 2) {
              if (m >= nm) break;
              const uint32_t a0 = sa + ra[m] * 128u, x0 = ra[m] & 7u;
              const uint32_t b0 = sb + rbv[m] * 128u, y0 = rbv[m] & 7u;
              float u0 = acc[m];
              if (m + 1 < nm) {
                const uint32_t a1 = sa + ra[m + 1] * 128u, x1 = ra[m + 1] & 7u;
                const uint32_t b1 = sb + rbv[m + 1] * 128u, y1 = rbv[m + 1] & 7u;
                float u1 = acc[m + 1];
#pragma unroll
                for (int g = 0; g < kRcKC / 4; g++) {
                  const float4 pa = lds4(a0 + ((g ^ x0) << 4)), pbv = lds4(b0 + ((g ^ y0) << 4));
                  const float4 qa = lds4(a1 + ((g ^ x1) << 4)), qb = lds4(b1 + ((g ^ y1) << 4));
                  u0 = __fmaf_rn(pa.x, pbv.x, u0);
                  u1 = __fmaf_rn(qa.x, qb.x, u1);
                  u0 = __fmaf_rn(pa.y, pbv.y, u0);
                  u1 = __fmaf_rn(qa.y, qb.y, u1);
                  u0 = __fmaf_rn(pa.z, pbv.z, u0);
                  u1 = __fmaf_rn(qa.z, qb.z, u1);
                  u0 = __fmaf_rn(pa.w, pbv.w, u0);
                  u1 = __fmaf_rn(qa.w, qb.w, u1);
                }
                acc[m + 1] = u1;
              } else {
#pragma unroll
                for (int g = 0; g < kRcKC / 4; g++) {
                  const float4 pa = lds4(a0 + ((g ^ x0) << 4)), pbv = lds4(b0 + ((g ^ y0) << 4));
                  u0 = __fmaf_rn(pa.x, pbv.x, u0);
                  u0 = __fmaf_rn(pa.y, pbv.y, u0);
                  u0 = __fmaf_rn(pa.z, pbv.z, u0);
                  u0 = __fmaf_rn(pa.w, pbv.w, u0);
                }
              }
              acc[m] = u0;
            }
          } else {
#pragma unroll
            for (int m = 0; m < kRtCpt; m++) {
              if (m >= nm) break;
              float u0 = acc[m];
              for (int e = 0; e < kc; e++)
                u0 = __fmaf_rn(lds1(sa + swz(ra[m], e)), lds1(sb + swz(rbv[m], e)), u0);
              acc[m] = u0;
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_relaxed(&empty[s]);
          if (++s == kRtStages) {
            s = 0;
            ph ^= 1u;
          }
        }
#pragma unroll
        for (int m = 0; m < kRtCpt; m++)
          if (m < nm)
            finish_candidate(sims, pb + ct + m * kCT, r0 + ra[m], acc[m], theta, p.rowcount);
      }
    }
  }
}

// --------------------------------------- recheck, tile groups, A reused
// recheck_tma_kernel streams the R-block (A) chunks again for every tile,
// although all tiles of a work item share the R block: its shared-memory
// traffic per tile is 24 x (32 KB A + 32 KB B written) + the operand reads.
// Here consecutive tiles of an item form a group whose candidates fit in
// shared memory (<= kGrCap): per K chunk the A chunk is staged once for the
// group and the B chunk once per tile, and each candidate's fp32 running sum
// stays in shared memory between chunks (same d = 0..dim-1 order).  A tile
// with more candidates than the capacity runs alone, in passes.
constexpr int kGrCap = 8192;        // candidates per group
constexpr int kGrAStages = 2;
constexpr int kGrBStages = 3;
constexpr int kGrQ = 4;             // item queue slots (producer -> compute warps)

__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kRtComputeWarps * 32) : "memory");
}

__host__ __device__ constexpr uint32_t recheck_group_smem_bytes() {
  return (kGrAStages + kGrBStages) * kRtOpBytes + 1024 + kGrCap * 4 + kGrCap * 2 +
         2 * (kGrAStages + kGrBStages) * 8 + 3 * kGrQ * 8 + 64;
}

// Group [k, kend) of an item's tiles (local tile indices into toff), or one
// oversized tile k processed in passes.  Deterministic: the producer and
// the consumers walk identical groups.
__device__ __forceinline__ int64_t group_end(const uint32_t* toff, int64_t k, int64_t k_end) {
  const uint32_t g_lo = toff[k];
  int64_t e = k;
  while (e < k_end && toff[e + 1] - g_lo <= (uint32_t)kGrCap) e++;
  return e == k ? k + 1 : e;
}

// Where the filter put an item's candidates: it ran item i on CTA i % G as
// that CTA's (i / G)-th item, recording each of its tiles' first slot in
// toff (local tile index = tiles of the CTA's earlier items; every S chunk
// but the last has tiles_per_chunk tiles).
struct ItemLoc {
  int64_t owner, k, k_end, t0;
};
__device__ __forceinline__ ItemLoc item_loc(const RecheckParams& p, int64_t item) {
  const int G = p.filter_grid, nb = p.n_ablk, tpc = p.tiles_per_chunk;
  const int64_t n_chunks = p.n_items / nb;
  const int64_t last_tiles =
      mn<int64_t>(tpc, p.n_btiles - (p.tile_begin + (n_chunks - 1) * (int64_t)tpc));
  const int64_t c = item % G, m = item / G;
  const int64_t n_full = p.n_items - nb;  // items of every chunk but the last
  const int64_t cf = n_full > c ? (n_full - c + G - 1) / G : 0;
  ItemLoc L;
  L.owner = c;
  L.k = m <= cf ? m * tpc : cf * tpc + (m - cf) * last_tiles;
  const int64_t sc = item / nb;
  L.t0 = p.tile_begin + sc * tpc;
  const int64_t t1 = mn<int64_t>(L.t0 + tpc, p.n_btiles);
  L.k_end = L.k + (t1 - L.t0);
  return L;
}

// Items are handed out dynamically (one global counter, S-chunk-major order
// like the filter), so the CTAs stay within a couple of S chunks of each
// other however uneven the candidate counts are and the staged S rows are
// L2 hits; the filter's static item -> CTA assignment let fast CTAs run
// many chunks ahead and re-read S from DRAM (~23x at the cfg4 shape).
__global__ void __launch_bounds__(kRtThreads, 1)
    recheck_group_kernel(const __grid_constant__ RecheckTmaParams tp) {
  const RecheckParams& p = tp.b;
  extern __shared__ uint8_t rg_raw[];
  const uint32_t raw = smem_u32(rg_raw);
  uint8_t* base = rg_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* a_ring = base;                                        // kGrAStages x 32 KB
  uint8_t* b_ring = base + kGrAStages * kRtOpBytes;              // kGrBStages x 32 KB
  float* acc = reinterpret_cast<float*>(base + (kGrAStages + kGrBStages) * kRtOpBytes);
  uint16_t* meta = reinterpret_cast<uint16_t*>(acc + kGrCap);   // ra | rb << 8
  uint64_t* full_a = reinterpret_cast<uint64_t*>(meta + kGrCap);
  uint64_t* empty_a = full_a + kGrAStages;
  uint64_t* full_b = empty_a + kGrAStages;
  uint64_t* empty_b = full_b + kGrBStages;
  uint64_t* item_full = empty_b + kGrBStages;
  uint64_t* item_empty = item_full + kGrQ;
  volatile int64_t* items = reinterpret_cast<volatile int64_t*>(item_empty + kGrQ);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kGrAStages; i++) {
      mbar_init(&full_a[i], 1);
      mbar_init(&empty_a[i], kRtComputeWarps);
    }
    for (int i = 0; i < kGrBStages; i++) {
      mbar_init(&full_b[i], 1);
      mbar_init(&empty_b[i], kRtComputeWarps);
    }
    for (int i = 0; i < kGrQ; i++) {
      mbar_init(&item_full[i], 1);
      mbar_init(&item_empty[i], kRtComputeWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int dim = p.dim;
  const int nch = (dim + kRcKC - 1) / kRcKC;
  const int nb = p.n_ablk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int sa = 0, sbs = 0, qs = 0;
  uint32_t pha = 0, phb = 0, qph = 0;

  if (warp == 0) {
    if (lane != 0) return;
    // -------------------------------------------------------- producer
    for (;;) {
      int64_t item = (int64_t)atomicAdd(p.work, 1u);
      if (item >= p.n_items) item = -1;
      mbar_wait(&item_empty[qs], qph ^ 1u);
      items[qs] = item;
      mbar_arrive(&item_full[qs]);
      if (++qs == kGrQ) { qs = 0; qph ^= 1u; }
      if (item < 0) break;
      const ItemLoc L = item_loc(p, item);
      if (p.cta_count[L.owner] > p.seg_cap) continue;  // saturated segment: the join is retried
      const uint32_t* toff = p.tile_off + L.owner * p.tile_stride;
      const int64_t rb = item % nb;
      for (int64_t kg = L.k; kg < L.k_end;) {
        const int64_t ke = group_end(toff, kg, L.k_end);
        const uint32_t g_lo = toff[kg], g_hi = toff[ke];
        if (g_hi - g_lo >= p.direct_max) {
          for (uint32_t pb = g_lo; pb < g_hi; pb += kGrCap) {   // > 1 pass: one oversized tile
            for (int ch = 0; ch < nch; ch++) {
              mbar_wait(&empty_a[sa], pha ^ 1u);
              mbar_arrive_expect_tx(&full_a[sa], kRtOpBytes);
              tma2d(a_ring + (size_t)sa * kRtOpBytes, &tp.tmap_l, ch * kRcKC,
                    (int)(rb * kTileRows), &full_a[sa]);
              if (++sa == kGrAStages) { sa = 0; pha ^= 1u; }
              for (int64_t kt = kg; kt < ke; kt++) {
                if (toff[kt + 1] == toff[kt]) continue;
                mbar_wait(&empty_b[sbs], phb ^ 1u);
                mbar_arrive_expect_tx(&full_b[sbs], kRtOpBytes);
                tma2d(b_ring + (size_t)sbs * kRtOpBytes, &tp.tmap_r, ch * kRcKC,
                      (int)((L.t0 + (kt - L.k)) * kTileRows), &full_b[sbs]);
                if (++sbs == kGrBStages) { sbs = 0; phb ^= 1u; }
              }
            }
          }
        }
        kg = ke;
      }
    }
    return;
  }
  // ------------------------------------------------------------ compute
  const int ct = threadIdx.x - 32;
  constexpr int kCT = kRtComputeWarps * 32;
  const float theta = p.theta;
  for (;;) {
    mbar_wait(&item_full[qs], qph);
    const int64_t item = items[qs];
    __syncwarp();
    if (lane == 0) mbar_arrive_relaxed(&item_empty[qs]);
    if (++qs == kGrQ) { qs = 0; qph ^= 1u; }
    if (item < 0) break;
    const ItemLoc L = item_loc(p, item);
    if (p.cta_count[L.owner] > p.seg_cap) continue;
    const uint64_t* seg = p.cand + (uint64_t)L.owner * p.seg_cap;
    uint32_t* sims = p.sims_bits + (uint64_t)L.owner * p.seg_cap;
    const uint32_t* toff = p.tile_off + L.owner * p.tile_stride;
    for (int64_t kg = L.k; kg < L.k_end;) {
      const int64_t ke = group_end(toff, kg, L.k_end);
      const uint32_t g_lo = toff[kg], g_hi = toff[ke];
      if (g_hi - g_lo < p.direct_max) {
        for (uint32_t q = g_lo + ct; q < g_hi; q += kCT) {   // few candidates: gather
          const uint64_t u = seg[q];
          const uint32_t gi = (uint32_t)(u >> 32), gj = (uint32_t)u;
          const float x = dot_seq_dev(p.l32 + (size_t)gi * dim, p.r32 + (size_t)gj * dim, dim);
          finish_candidate(sims, q, gi, x, theta, p.rowcount);
        }
        kg = ke;
        continue;
      }
      for (uint32_t pb = g_lo; pb < g_hi; pb += kGrCap) {
        const uint32_t np = mn<uint32_t>(g_hi - pb, (uint32_t)kGrCap);
        consumer_bar();   // the previous pass's finish has read acc / meta
        for (uint32_t q = ct; q < np; q += kCT) {
          const uint64_t u = seg[pb + q];
          meta[q] = (uint16_t)(((uint32_t)(u >> 32) & 255u) | (((uint32_t)u & 255u) << 8));
          acc[q] = 0.0f;
        }
        consumer_bar();
        for (int ch = 0; ch < nch; ch++) {
          mbar_wait(&full_a[sa], pha);
          const uint32_t sA = smem_u32(a_ring + (size_t)sa * kRtOpBytes);
          const int kc = mn(kRcKC, dim - ch * kRcKC);
          for (int64_t kt = kg; kt < ke; kt++) {
            const uint32_t lo = toff[kt], hi = toff[kt + 1];
            if (hi == lo) continue;
            mbar_wait(&full_b[sbs], phb);
            const uint32_t sB = smem_u32(b_ring + (size_t)sbs * kRtOpBytes);
            // this pass's positions of tile kt
            const uint32_t ps = (lo > pb ? lo : pb) - pb, pe = mn<uint32_t>(hi, pb + np) - pb;
            for (uint32_t q = ps + ct; q < pe; q += kCT) {
              const uint32_t m = meta[q], ra = m & 255u, rbv = m >> 8;
              float x = acc[q];
              if (kc == kRcKC) {
                const uint32_t a0 = sA + ra * 128u, xa = ra & 7u;
                const uint32_t b0 = sB + rbv * 128u, yb = rbv & 7u;
#pragma unroll
                for (int g = 0; g < kRcKC / 4; g++) {
                  const float4 va = lds4(a0 + ((g ^ xa) << 4)), vb = lds4(b0 + ((g ^ yb) << 4));
                  x = __fmaf_rn(va.x, vb.x, x);
                  x = __fmaf_rn(va.y, vb.y, x);
                  x = __fmaf_rn(va.z, vb.z, x);
                  x = __fmaf_rn(va.w, vb.w, x);
                }
              } else {
                for (int e = 0; e < kc; e++) x = __fmaf_rn(lds1(sA + swz(ra, e)), lds1(sB + swz(rbv, e)), x);
              }
              acc[q] = x;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&empty_b[sbs]);
            if (++sbs == kGrBStages) { sbs = 0; phb ^= 1u; }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_relaxed(&empty_a[sa]);
          if (++sa == kGrAStages) { sa = 0; pha ^= 1u; }
        }
        consumer_bar();   // every chunk of every position done
        for (uint32_t q = ct; q < np; q += kCT) {
          const uint64_t u = seg[pb + q];
          finish_candidate(sims, pb + q, (uint32_t)(u >> 32), acc[q], theta, p.rowcount);
        }
      }
      kg = ke;
    }
  }
}

// Canonical recheck of the pending pairs of tolerance emission (the pairs
// within the band of theta; everything else was decided by the filter).
// Pending entry k of CTA c is visited at position p = k * grid + c, so
// neighbouring threads work on pairs the filter emitted at about the same
// time -- from the same few S chunks, which are then L2 hits.  Two
// independent sequential chains per thread (dot_seq2_dev, bitwise
// sj_dot_seq).  Saturated segments are skipped: the join is retried.
__global__ void __launch_bounds__(256)
recheck_pending_kernel(const uint64_t* __restrict__ cand, uint64_t seg_cap,
                       const uint32_t* __restrict__ pend, const uint32_t* __restrict__ pend_count,
                       const unsigned long long* __restrict__ cta_count, int n_cta,
                       const float* __restrict__ l32, const float* __restrict__ r32, int dim,
                       float theta, uint32_t* __restrict__ sims_bits,
                       uint32_t* __restrict__ rowcount) {
  __shared__ uint32_t s_max;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < n_cta; c += blockDim.x) atomicMax(&s_max, pend_count[c]);
  __syncthreads();
  const uint64_t total = (uint64_t)s_max * (uint64_t)n_cta;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  auto locate = [&](uint64_t p, uint64_t* slot, uint32_t* gi, uint32_t* gj) -> bool {
    if (p >= total) return false;
    const uint64_t k = p / (uint64_t)n_cta, c = p - k * (uint64_t)n_cta;
    if (k >= pend_count[c] || cta_count[c] > seg_cap) return false;
    *slot = c * seg_cap + pend[c * seg_cap + k];
    const uint64_t u = cand[*slot];
    *gi = (uint32_t)(u >> 32);
    *gj = (uint32_t)u;
    return true;
  };
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < total; p += 2 * stride) {
    uint64_t s0 = 0, s1 = 0;
    uint32_t i0 = 0, j0 = 0, i1 = 0, j1 = 0;
    const bool a = locate(p, &s0, &i0, &j0);
    const bool b = locate(p + stride, &s1, &i1, &j1);
    if (a && b) {
      float x0, x1;
      dot_seq2_dev(l32 + (size_t)i0 * dim, r32 + (size_t)j0 * dim, l32 + (size_t)i1 * dim,
                   r32 + (size_t)j1 * dim, dim, x0, x1);
      finish_candidate(sims_bits, s0, i0, x0, theta, rowcount);
      finish_candidate(sims_bits, s1, i1, x1, theta, rowcount);
    } else if (a) {
      finish_candidate(sims_bits, s0, i0, dot_seq_dev(l32 + (size_t)i0 * dim, r32 + (size_t)j0 * dim, dim),
                       theta, rowcount);
    } else if (b) {
      finish_candidate(sims_bits, s1, i1, dot_seq_dev(l32 + (size_t)i1 * dim, r32 + (size_t)j1 * dim, dim),
                       theta, rowcount);
    }
  }
}

// The same recheck with the rows STAGED: a warp takes 32 consecutive positions
// (lane = pair) and walks both rows of every pair in 32-element chunks.  The
// whole warp copies a chunk of all 64 rows with 16-byte cp.async (8 lanes per
// 128-byte line: full sectors, coalesced) into its shared-memory ring, and each
// lane then advances its own pair's chain from shared memory (16-byte pieces
// XOR-swizzled by the pair index: conflict-free for lane = row reads).  The
// thread-per-pair gather above touches 32 different sectors per load
// instruction and re-fetches each sector's other half from L2 once the SM's
// 2048 threads' working set outgrows L1; this kernel moves each row byte once.
// dim % 4 = 0 and 16-byte aligned rows (the caller checks).
constexpr int kPsWarps = 8;
constexpr int kPsBufs = 3;                       // chunks in the ring (two in flight)
constexpr int kPsChunk = 32;                     // elements per chunk (128 B per row)
constexpr uint32_t kPsBufBytes = 2u * 32u * kPsChunk * 4u;   // 32 pairs x 2 rows
__host__ __device__ constexpr uint32_t pending_staged_smem() {
  return kPsWarps * kPsBufs * kPsBufBytes;
}

__device__ __forceinline__ void cp_async_wait_two() { asm volatile("cp.async.wait_group 2;" ::: "memory"); }

__global__ void __launch_bounds__(kPsWarps * 32, 1)
recheck_pending_staged_kernel(const uint64_t* __restrict__ cand, uint64_t seg_cap,
                              const uint32_t* __restrict__ pend,
                              const uint32_t* __restrict__ pend_count,
                              const unsigned long long* __restrict__ cta_count, int n_cta,
                              const float* __restrict__ l32, const float* __restrict__ r32, int dim,
                              float theta, uint32_t* __restrict__ sims_bits,
                              uint32_t* __restrict__ rowcount) {
  extern __shared__ __align__(128) uint8_t ps_smem[];
  __shared__ uint32_t s_max;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < n_cta; c += blockDim.x) atomicMax(&s_max, pend_count[c]);
  __syncthreads();
  const uint64_t total = (uint64_t)s_max * (uint64_t)n_cta;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = ps_smem + (size_t)warp * kPsBufs * kPsBufBytes;
  const int nchunks = (dim + kPsChunk - 1) / kPsChunk;
  const int sub = lane >> 3, piece = lane & 7;   // this lane's share of every copy round
  const uint64_t n_groups = (total + 31) / 32;
  for (uint64_t g = (uint64_t)blockIdx.x * kPsWarps + warp; g < n_groups;
       g += (uint64_t)gridDim.x * kPsWarps) {
    const uint64_t p = g * 32 + lane;
    bool ok = false;
    uint64_t slot = 0;
    uint32_t gi = 0, gj = 0;
    if (p < total) {
      const uint64_t k = p / (uint64_t)n_cta, c = p - k * (uint64_t)n_cta;
      if (k < pend_count[c] && cta_count[c] <= seg_cap) {
        slot = c * seg_cap + pend[c * seg_cap + k];
        const uint64_t u = cand[slot];
        gi = (uint32_t)(u >> 32);
        gj = (uint32_t)u;
        ok = true;
      }
    }
    if (!__any_sync(0xffffffffu, ok)) continue;
    // the 8 pairs whose lines this lane copies in every chunk: sub, sub + 4, ...
    const float* srcA[8];
    const float* srcB[8];
#pragma unroll
    for (int it = 0; it < 8; it++) {
      const uint32_t i = __shfl_sync(0xffffffffu, gi, it * 4 + sub);
      const uint32_t j = __shfl_sync(0xffffffffu, gj, it * 4 + sub);
      srcA[it] = l32 + (size_t)i * dim + piece * 4;
      srcB[it] = r32 + (size_t)j * dim + piece * 4;
    }
    auto issue = [&](int c) {
      if (c < nchunks && c * kPsChunk + piece * 4 < dim) {
        uint8_t* buf = ring + (size_t)(c % kPsBufs) * kPsBufBytes;
#pragma unroll
        for (int it = 0; it < 8; it++) {
          const int pr = it * 4 + sub;
          const uint32_t off = (uint32_t)pr * 128u + (uint32_t)((piece ^ (pr & 7)) * 16);
          cp_async16(reinterpret_cast<float*>(buf + off), srcA[it] + c * kPsChunk);
          cp_async16(reinterpret_cast<float*>(buf + 4096u + off), srcB[it] + c * kPsChunk);
        }
      }
      cp_async_commit();
    };
    issue(0);
    issue(1);
    float acc = 0.0f;
    for (int c = 0; c < nchunks; c++) {
      issue(c + 2);
      cp_async_wait_two();   // chunk c has landed (this lane's copies)
      __syncwarp();          // ... and every lane's
      const uint8_t* buf = ring + (size_t)(c % kPsBufs) * kPsBufBytes + (uint32_t)lane * 128u;
      const int np = mn<int>(8, (dim - c * kPsChunk) >> 2);
#pragma unroll
      for (int q = 0; q < 8; q++) {
        if (q < np) {
          const uint32_t o = (uint32_t)((q ^ (lane & 7)) * 16);
          const float4 x = *reinterpret_cast<const float4*>(buf + o);
          const float4 y = *reinterpret_cast<const float4*>(buf + 4096u + o);
          acc = __fmaf_rn(x.x, y.x, acc);
          acc = __fmaf_rn(x.y, y.y, acc);
          acc = __fmaf_rn(x.z, y.z, acc);
          acc = __fmaf_rn(x.w, y.w, acc);
        }
      }
      __syncwarp();          // the buffer may be refilled (chunk c + 3)
    }
    if (ok) finish_candidate(sims_bits, slot, gi, acc, theta, rowcount);
  }
}

// Canonical recheck of every candidate of the CTA-pair filter's segments
// (canonical sims on raw operands, SJB_WIDE_EXACT=rows), in the FILTER'S ORDER:
// recheck CTA c walks segment c from its start, so all CTAs stay on the S chunk
// the filter CTAs were on together and the S rows are L2 hits (grouping the
// candidates by left row first was measured: the recheck turned DRAM-bound,
// 27.5 ms at the cfg4 slice).  Row sharing is recovered locally: a block of
// 2048 consecutive candidates (half a work item: 128 left rows, ~16
// candidates each at cfg4) is counting-sorted by left row in shared memory,
// and a warp then takes 32 neighbours of that order -- 2-3 distinct left rows
// -- and stages each DISTINCT left row once (the lanes of a row read its
// leader's copy: a broadcast) beside the 32 private S rows, with the ring,
// swizzle and chain of recheck_pending_staged_kernel.  A candidate moves
// ~4 d bytes from L2 instead of 8 d.  sims_bits[slot] gets the canonical bits
// or kRejected; kept matches are counted per left row.
constexpr int kRsBlock = 2048;
// ring stage: 8 shared left-row slots (1 KB) + the 32 private S rows (4 KB); 5 stages, four
// chunks in flight per warp.  (With the 8 KB stages and 3-deep ring of the pending kernel this
// kernel ran at ~7 TB/s of L2 -> SM traffic: 72 KB in flight per SM against ~2000 cycles of
// loaded L2 latency.  The staged kernels are bound by bytes in flight, not by bandwidth.)
constexpr int kRsLead = 8;
constexpr int kRsBufs = 5;
constexpr uint32_t kRsABytes = kRsLead * 128u;
constexpr uint32_t kRsBufBytes = kRsABytes + 32u * 128u;
constexpr uint32_t kRsRingBytes = kPsWarps * kRsBufs * kRsBufBytes;
__host__ __device__ constexpr uint32_t recheck_sorted_smem() {
  return kRsRingBytes + kRsBlock * 8 + kRsBlock * 2 + 2 * 256 * 4 + 64;
}
__device__ __forceinline__ void cp_async_wait_four() { asm volatile("cp.async.wait_group 4;" ::: "memory"); }

// Work units (pair work item, CTA of the pair) are handed out by a counter in the
// filter's S-chunk-major item order, so every recheck CTA is on the same few S chunks
// (walking the segments by position lets them drift chunks apart: the S rows then come
// from DRAM); the unit's candidates are segment [toff[k], toff[k + 1]) of its filter CTA.
__global__ void __launch_bounds__(kPsWarps * 32, 1)
recheck_segments_sorted_kernel(const uint64_t* __restrict__ cand, uint64_t seg_cap,
                               const unsigned long long* __restrict__ cta_count,
                               const uint32_t* __restrict__ tile_off, int64_t tile_stride,
                               int64_t n_items, int n_pairs, unsigned int* __restrict__ work,
                               const float* __restrict__ l32, const float* __restrict__ r32,
                               int dim, float theta, uint32_t* __restrict__ sims_bits,
                               uint32_t* __restrict__ rowcount) {
  extern __shared__ __align__(128) uint8_t ps_smem[];
  __shared__ unsigned int s_unit;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* ring = ps_smem + (size_t)warp * kRsBufs * kRsBufBytes;
  uint64_t* sorted = reinterpret_cast<uint64_t*>(ps_smem + kRsRingBytes);
  uint16_t* sidx = reinterpret_cast<uint16_t*>(sorted + kRsBlock);
  uint32_t* hist = reinterpret_cast<uint32_t*>(sidx + kRsBlock);   // [256] counts, then cursors
  uint32_t* wtot = hist + 256;                                      // [8] warp totals
  const int nchunks = (dim + kPsChunk - 1) / kPsChunk;
  const int sub = lane >> 3, piece = lane & 7;
  for (;;) {
  if (tid == 0) s_unit = atomicAdd(work, 1u);
  __syncthreads();
  const int64_t unit = (int64_t)s_unit;
  __syncthreads();
  if (unit >= 2 * n_items) break;
  const int64_t item = unit >> 1;
  const int fc = 2 * (int)(item % n_pairs) + (int)(unit & 1);   // the filter CTA
  const int64_t k = item / n_pairs;                             // its k-th work item
  if (cta_count[fc] > seg_cap) continue;   // saturated segment: the join is retried with room
  const uint64_t* seg = cand + (uint64_t)fc * seg_cap;
  uint32_t* sims = sims_bits + (uint64_t)fc * seg_cap;
  const uint32_t* toff = tile_off + (int64_t)fc * tile_stride;
  const uint64_t lo = toff[k], cc = toff[k + 1];
  for (uint64_t b0 = lo; b0 < cc; b0 += kRsBlock) {
    const int nb = (int)mn<uint64_t>(kRsBlock, cc - b0);
    // ---- counting sort of the block by (left row & 255)
    hist[tid] = 0u;   // 256 threads
    __syncthreads();
    for (int t = tid; t < nb; t += kPsWarps * 32)
      atomicAdd(&hist[(uint32_t)(seg[b0 + t] >> 32) & 255u], 1u);
    __syncthreads();
    {
      const uint32_t v = hist[tid];
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wtot[warp] = incl;
      __syncthreads();
      uint32_t base = 0;
      for (int w = 0; w < warp; w++) base += wtot[w];
      hist[tid] = base + incl - v;   // exclusive prefix: the bucket's cursor
    }
    __syncthreads();
    for (int t = tid; t < nb; t += kPsWarps * 32) {
      const uint64_t u = seg[b0 + t];
      const uint32_t pos = atomicAdd(&hist[(uint32_t)(u >> 32) & 255u], 1u);
      sorted[pos] = u;
      sidx[pos] = (uint16_t)t;
    }
    __syncthreads();
    // ---- staged recheck of 32 neighbours of the sorted order per warp
    for (int e0 = warp * 32; e0 < nb; e0 += kPsWarps * 32) {
      const int e = e0 + lane;
      const bool ok = e < nb;
      uint32_t gi = 0, gj = 0, slot = 0;
      if (ok) {
        const uint64_t u = sorted[e];
        gi = (uint32_t)(u >> 32);
        gj = (uint32_t)u;
        slot = (uint32_t)sidx[e];
      }
      // passes of <= kRsLead distinct left rows (one pass unless the warp's candidates
      // are spread over more rows: sparse joins)
      uint32_t todo = __ballot_sync(0xffffffffu, ok);
      while (todo) {
        const bool mine = (todo >> lane) & 1u;
        // a lane's left row is staged by its leader: the first pending lane with the same row
        const uint32_t same = __match_any_sync(0xffffffffu, mine ? gi : 0xFFFFFFFFu) & todo;
        const int leader = mine ? __ffs(same) - 1 : lane;
        const uint32_t lead_mask = __ballot_sync(0xffffffffu, mine && leader == lane);
        const uint32_t rank = __popc(lead_mask & ((1u << leader) - 1u));   // the leader's A slot
        const bool active = mine && rank < (uint32_t)kRsLead;
        const uint32_t act_mask = __ballot_sync(0xffffffffu, active);
        const float* srcA[8];
        const float* srcB[8];
        uint32_t offA[8];
#pragma unroll
        for (int it = 0; it < 8; it++) {
          const int pr = it * 4 + sub;
          const uint32_t i = __shfl_sync(0xffffffffu, gi, pr);
          const uint32_t j = __shfl_sync(0xffffffffu, gj, pr);
          srcA[it] = l32 + (size_t)i * dim + piece * 4;
          srcB[it] = r32 + (size_t)j * dim + piece * 4;
          const uint32_t rk = __popc(lead_mask & ((1u << pr) - 1u));
          // leaders of active groups copy their left row into slot rk
          offA[it] = ((lead_mask & act_mask) >> pr) & 1u
                         ? rk * 128u + (uint32_t)((piece ^ (int)(rk & 7u)) * 16)
                         : 0xFFFFFFFFu;
        }
        auto issue = [&](int c) {
          if (c < nchunks && c * kPsChunk + piece * 4 < dim) {
            uint8_t* buf = ring + (size_t)(c % kRsBufs) * kRsBufBytes;
#pragma unroll
            for (int it = 0; it < 8; it++) {
              const int pr = it * 4 + sub;
              if (offA[it] != 0xFFFFFFFFu)
                cp_async16(reinterpret_cast<float*>(buf + offA[it]), srcA[it] + c * kPsChunk);
              if ((act_mask >> pr) & 1u)
                cp_async16(reinterpret_cast<float*>(buf + kRsABytes + (uint32_t)pr * 128u +
                                                    (uint32_t)((piece ^ (pr & 7)) * 16)),
                           srcB[it] + c * kPsChunk);
            }
          }
          cp_async_commit();
        };
        issue(0);
        issue(1);
        issue(2);
        issue(3);
        float acc = 0.0f;
        const uint32_t a_row = (rank & 7u) * 128u, a_swz = rank & 7u;
        for (int c = 0; c < nchunks; c++) {
          issue(c + 4);
          cp_async_wait_four();
          __syncwarp();
          const uint8_t* buf = ring + (size_t)(c % kRsBufs) * kRsBufBytes;
          const int np = mn<int>(8, (dim - c * kPsChunk) >> 2);
#pragma unroll
          for (int q = 0; q < 8; q++) {
            if (q < np) {
              const float4 x =
                  *reinterpret_cast<const float4*>(buf + a_row + (((uint32_t)q ^ a_swz) * 16u));
              const float4 y = *reinterpret_cast<const float4*>(
                  buf + kRsABytes + (uint32_t)lane * 128u + (uint32_t)((q ^ (lane & 7)) * 16));
              acc = __fmaf_rn(x.x, y.x, acc);
              acc = __fmaf_rn(x.y, y.y, acc);
              acc = __fmaf_rn(x.z, y.z, acc);
              acc = __fmaf_rn(x.w, y.w, acc);
            }
          }
          __syncwarp();
        }
        const bool keep = active && acc >= theta;
        if (active) sims[b0 + slot] = keep ? __float_as_uint(acc) : kRejected;
        // one atomic per distinct left row of the pass
        const uint32_t kept = __popc(__ballot_sync(0xffffffffu, keep) & same);
        if (active && leader == lane && kept) atomicAdd(rowcount + gi, kept);
        todo &= ~act_mask;
      }
    }
    __syncthreads();   // the block's buffers are reused
  }
  }
}

}  // namespace wide
}  // namespace sjb
