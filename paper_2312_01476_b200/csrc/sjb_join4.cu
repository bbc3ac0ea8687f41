// sjb_join4.cu -- the K-streaming (d > 128) filter on CTA PAIRS (cta_group::2),
// tolerance emission (raw bf16 operands, tensor similarities; BASELINE cfg4).
// The default filter of that mode (kTwo = true).
//
// The 1-CTA wide filter (sjb_join3.cu) computes a 256 x 256 output tile per SM
// and that tile fills the SM's tensor memory (2 x 256 columns), so there is no
// second accumulator: after a tile's last MMA the tensor pipe waits until the
// epilogue has drained, normalised and emitted most of the tile.  At the cfg4
// selectivity (4e-3: 98% of the 32 x 64 warp chunks hold a candidate) that is
// ~45% of the tile's time: `tools/wide_modes.py` on a 16k x 1M slice gives
// filter 22.0 ms, tensor pipe 51% active, against 14.9 ms / 95% with the
// epilogue switched off -- operand delivery is NOT the limit.
//
// A pair of SMs sharing one UMMA (cta_group::2, M = 256 across the pair) halves
// the accumulator per SM: each CTA holds 128 rows of the R block (its M half)
// and 128 rows of the S tile (its half of the N = 256 operand), and gets 128
// lanes x 256 columns of the 256 x 256 pair tile -- HALF its tensor memory.
// The other half is a second accumulator stage: the pair's MMAs run on tile
// t + 1 while both CTAs drain tile t (kTwo).  Operand bytes per MMA and per SM
// are those of the 1-CTA kernel (32 KB per 512 MMA cycles).  With 16 epilogue
// warps on 32-column chunks (90 registers, four warps per scheduler to hide the
// emission's latencies) the same slice's filter takes 15.2 ms, tensor pipe 97%
// active (8 warps on 64-column chunks: 17.0 ms, 79%).
//
//   * TMEM per CTA: 128 lanes (its R rows) x 2 stages x 256 columns.
//   * Operands: 3-D tensor TMA (.cta_group::2, completing on the leader's
//     barrier) of the [k-group][row][8] operand image: box {256, 4, 8} =
//     [8 k-groups][128 rows][8] of one image tile = 16 KB, the UMMA K-major
//     layout (k-group stride 2 KB).  Two per CTA per K chunk: its R half and
//     its 128-row half of the S tile.
//   * The leader's warp 1 issues every MMA of the pair; commits are multicast
//     to both CTAs (ring slots, accumulator full); the epilogue warps of both
//     CTAs arrive on the leader's accumulator-empty barriers.
//   * Epilogue: normalise after the GEMM (the tile's inverse norms prefetched
//     per warp into shared memory before the accumulator wait), then the
//     tolerance emission (final / pending / no candidate) per chunk.
//
// kTwo = false (A/B build, SJB_WIDE_MMA2=1) is the first form tried: a 256 x 512
// pair tile in one accumulator (each CTA: 128 x 512 outputs per 48 KB per K
// chunk, 25% fewer operand bytes) -- no faster than the 1-CTA kernel, which is
// what showed the operand stream was not the limit.
#include "sjb_common.cuh"

namespace sjb {
namespace wide2 {

constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clears the CTA-rank bit of a pair smem address

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// relaxed arrive on the barrier at the same offset in the leader CTA
__device__ __forceinline__ void arrive_leader_relaxed(uint64_t* bar) {
  const uint32_t a = smem_u32(bar) & kPeerMask;
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
// 3-D tensor TMA into this CTA's shared memory, completing on the leader's
// barrier (the address with the CTA-rank bit cleared)
__device__ __forceinline__ void tma3d_2sm(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                          uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1),
      "r"(c2), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// warp-uniform issue, one elected lane
__device__ __forceinline__ void mma2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                     uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit the pair's prior MMAs to the barrier at this offset in both CTAs
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

#ifndef SJB_WIDE2_EPI
#define SJB_WIDE2_EPI 16
#endif
// epilogue warps: 8 (64-column chunks) or 16 (32-column chunks: half the live
// accumulator registers per thread, four warps per scheduler to hide the
// emission's latencies)
constexpr int kEpiWarps = SJB_WIDE2_EPI;
static_assert(kEpiWarps == 8 || kEpiWarps == 16, "SJB_WIDE2_EPI: 8 or 16");
constexpr int kCW = kEpiWarps == 8 ? 64 : 32;   // columns per drained chunk
constexpr int kThreads = 32 * (2 + kEpiWarps);
// first column (within a 256-column accumulator half) of chunk k of the warps of column group cw
__device__ __forceinline__ int chunk_col(int cw, int k) {
  return kEpiWarps == 8 ? (cw + 2 * k) * 64 : cw * 64 + k * 32;
}
constexpr int kKChunk = 64;
constexpr int kHalfRows = 128;
constexpr uint32_t kPieceBytes = kHalfRows * kKChunk * 2;   // 16 KB
// ring stage: the R half + two S halves (256 x 512 pair tile, one accumulator
// tile), or -- kTwo -- the R half + one S half (256 x 256 pair tile, TWO
// accumulator stages of 256 columns: the drain of one tile overlaps the MMAs
// of the next; same operand bytes per MMA as the 1-CTA kernel)
__host__ __device__ constexpr uint32_t stage_bytes(bool two) {
  return (two ? 2u : 3u) * kPieceBytes;
}
constexpr int kTolPitch = 33;
constexpr uint32_t kTolScratchBytes = kEpiWarps * 32 * kTolPitch * 4;
// kTwo: each epilogue warp's copy of the tile's inverse norms of its two 64-column
// chunks (32 float4), prefetched before the accumulator wait: the normalisation reads
// them as shared-memory broadcasts instead of 16 L2-latency loads per chunk
constexpr uint32_t kInvStageBytes = kEpiWarps * 32 * 16;
__host__ __device__ constexpr int max_stages(bool two) {
  return (two ? 5 : 4) - (kEpiWarps == 16 ? 1 : 0);   // 16 warps: twice the emission scratch
}

struct alignas(64) Params {
  CUtensorMap tmap_a;   // R image as (256, 8, kgroups * tiles), box {256, 4, 8}
  CUtensorMap tmap_b;   // S image, same
  int64_t n_a, n_b;
  int kpad;
  int n_ablk;           // 256-row R tiles (one per pair)
  int n_ptiles;         // 512-row pair S tiles (kTwo: 256-row tiles) in this launch's range end
  int tiles_per_chunk;  // pair tiles per work item
  int tile_begin;       // first pair tile of this launch
  int append;
  int64_t n_items;      // pair items
  int stages;
  int bf16;
  float cutoff;
  float hi_cut;
  uint64_t* cand;
  uint64_t seg_cap;
  unsigned long long* cta_count;
  const float* inv_a;
  const float* inv_b;
  uint32_t* sims_bits;
  uint32_t* rowcount;
  uint32_t* pend;
  uint32_t* pend_count;
  uint32_t* tile_off;   // !tol: [grid][tile_stride] segment offset at each work item's start (+ end)
  int64_t tile_stride;
  int tol;     // 1: tolerance emission (tensor sims); 0: candidates only (canonical sims: the
               // row-grouped staged recheck decides every candidate afterwards)
  int debug;   // diagnostics (results invalid): 1 no emission, 2 no drain, 3 drain + normalise only,
               // 20 no operand traffic
};

__host__ __device__ inline uint32_t smem_bytes(int stages, bool two) {
  return (uint32_t)stages * stage_bytes(two) + (4 + 2 * stages) * 8 + 32 + kTolScratchBytes +
         (two ? kInvStageBytes : 0u);
}

template <bool kTwo>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    filter_kernel(const __grid_constant__ Params p) {
  constexpr uint32_t kStageBytes = stage_bytes(kTwo);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * kStageBytes);
  uint64_t* acc_full = bars + 0;    // [2] (kTwo: per accumulator stage), both: MMA commit (multicast)
  uint64_t* acc_empty = bars + 2;   // [2], leader: epilogue warps of both CTAs
  uint64_t* full = bars + 4;        // leader: the pair's operand bytes
  uint64_t* empty = bars + 4 + p.stages;   // both: MMA commit (multicast)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 + 2 * p.stages);
  uint32_t* cta_cnt = tmem_slot + 2;
  uint32_t* cta_sat = tmem_slot + 3;
  uint32_t* pend_cnt = tmem_slot + 5;
  float* tol_scratch = reinterpret_cast<float*>(tmem_slot + 8);
  float4* inv_stage = reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(tol_scratch) +
                                                kTolScratchBytes);   // kTwo only

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t pair_id = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    mbar_init(&acc_full[0], 1);
    mbar_init(&acc_full[1], 1);
    mbar_init(&acc_empty[0], 2 * kEpiWarps);
    mbar_init(&acc_empty[1], 2 * kEpiWarps);
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    init_segment_count(p.cta_count, p.append != 0, cta_cnt, cta_sat);
    *pend_cnt = 0u;
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t n_items = p.n_items;
  const int nb = p.n_ablk;
  const int nchunks = p.kpad / kKChunk;
  const int kg = p.kpad / 8;   // k-groups per image tile

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ producer (both CTAs)
      const uint64_t pol_a = policy_evict_last();
      const uint64_t pol_b = policy_evict_normal();
      int s = 0;
      uint32_t ph = 0;
      int64_t fills = 0;
      for (int64_t item = pair_id; item < n_items; item += n_pairs) {
        const int64_t rb = item % nb, sc = item / nb;
        const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_ptiles);
        for (int64_t t = t0; t < t1; t++) {
          for (int c = 0; c < nchunks; c++, fills++) {
            mbar_wait(&empty[s], ph ^ 1u);
            if (p.debug == 20 && fills >= p.stages) {   // diagnostics: no operand traffic
              if (leader) mbar_arrive(&full[s]);
              if (++s == p.stages) {
                s = 0;
                ph ^= 1u;
              }
              continue;
            }
            if (leader) mbar_arrive_expect_tx(&full[s], 2 * kStageBytes);
            uint8_t* dst = ring + (size_t)s * kStageBytes;
            tma3d_2sm(dst, &p.tmap_a, 0, 4 * (int)rank, (int)(rb * kg + c * 8), &full[s],
                            pol_a);
            if (kTwo) {
              tma3d_2sm(dst + kPieceBytes, &p.tmap_b, 0, 4 * (int)rank, (int)(t * kg + c * 8),
                        &full[s], pol_b);
            } else {
              tma3d_2sm(dst + kPieceBytes, &p.tmap_b, 0, 4 * (int)rank,
                        (int)(2 * t * kg + c * 8), &full[s], pol_b);
              tma3d_2sm(dst + 2 * kPieceBytes, &p.tmap_b, 0, 4 * (int)rank,
                        (int)((2 * t + 1) * kg + c * 8), &full[s], pol_b);
            }
            if (++s == p.stages) {
              s = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------- MMA issuer (the pair's)
      const uint32_t idesc = umma_idesc_f16_f32(256, 256, p.bf16 != 0);
      const uint32_t lbo = kHalfRows * 16, sbo = 128;
      const uint64_t kstep = (2 * lbo) >> 4;
      const uint64_t ring_desc = umma_desc_kmajor_noswz(smem_u32(ring), lbo, sbo);
      const uint64_t stage_step = kStageBytes >> 4, piece = kPieceBytes >> 4;
      int s = 0;
      uint32_t ph = 0, tile_it = 0;
      for (int64_t item = pair_id; item < n_items; item += n_pairs) {
        const int64_t sc = item / nb;
        const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_ptiles);
        for (int64_t t = t0; t < t1; t++, tile_it++) {
          for (int c = 0; c < nchunks; c++) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint64_t ad = ring_desc + (uint64_t)s * stage_step;
            if (kTwo) {
              const uint32_t st = tile_it & 1u;
              if (c == 0) {   // both CTAs drained the tile before last (same stage)?
                mbar_wait(&acc_empty[st], ((tile_it >> 1) & 1u) ^ 1u);
                tc_fence_after();
              }
              const uint64_t bd = ad + piece;
#pragma unroll
              for (int kk = 0; kk < kKChunk / 16; kk++)
                mma2(tmem_base + st * 256, ad + kk * kstep, bd + kk * kstep, idesc,
                     (c | kk) ? 1u : 0u);
            } else {
#pragma unroll
              for (int h = 0; h < 2; h++) {
                if (c == 0) {   // both CTAs drained half h of the previous tile?
                  mbar_wait(&acc_empty[h], (tile_it & 1u) ^ 1u);
                  tc_fence_after();
                }
                const uint64_t bd = ad + (uint64_t)(1 + h) * piece;
#pragma unroll
                for (int kk = 0; kk < kKChunk / 16; kk++)
                  mma2(tmem_base + h * 256, ad + kk * kstep, bd + kk * kstep, idesc,
                       (c | kk) ? 1u : 0u);
              }
            }
            commit2(&empty[s]);
            if (++s == p.stages) {
              s = 0;
              ph ^= 1u;
            }
          }
          commit2(&acc_full[kTwo ? (tile_it & 1u) : 0u]);
        }
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    // warp (q, c): TMEM lanes 32q..32q+31 (this CTA's R rows) x column
    // chunks c, c + 2 (64 each) of both halves; a half is handed back to the
    // leader after its last chunk is loaded
    const int ew = warp - 2;
    const int cw = ew >> 2, q = warp & 3;
    const uint32_t lane_base = (uint32_t)q * 32;
    uint64_t* seg = p.cand + (uint64_t)blockIdx.x * p.seg_cap;
    uint32_t* sims = p.sims_bits + (uint64_t)blockIdx.x * p.seg_cap;
    uint32_t* pend = p.pend + (uint64_t)blockIdx.x * p.seg_cap;
    float* scr = tol_scratch + (ew * 32 + lane) * kTolPitch;
    uint32_t tile_it = 0;
    uint32_t* toff = p.tol ? nullptr : p.tile_off + (int64_t)blockIdx.x * p.tile_stride;
    uint32_t item_k = 0;
    for (int64_t item = pair_id; item < n_items; item += n_pairs) {
      if (toff != nullptr) {
        // every epilogue warp is done with the previous item: the counter is this item's first slot
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        if (ew == 0 && lane == 0) toff[item_k] = *(volatile uint32_t*)cta_cnt;
        item_k++;
      }
      const int64_t rb = item % nb, sc = item / nb;
      const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
      const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_ptiles);
      const int64_t gi64 = rb * kTileRows + rank * kHalfRows + lane_base + lane;
      const bool row_ok = gi64 < p.n_a;
      const float inv_i = row_ok ? __ldg(p.inv_a + gi64) : 1.0f;
      uint32_t fin = 0u;
      for (int64_t t = t0; t < t1; t++, tile_it++) {
        float4 inv4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (kTwo && lane < 2 * (kCW / 4))   // the warp's two chunks' float4s; land during the wait
          inv4 = __ldg(reinterpret_cast<const float4*>(p.inv_b + t * kTileRows +
                                                       chunk_col(cw, lane / (kCW / 4))) +
                       (lane % (kCW / 4)));
        if (kTwo)
          mbar_wait(&acc_full[tile_it & 1u], (tile_it >> 1) & 1u);
        else
          mbar_wait(&acc_full[0], tile_it & 1u);
        tc_fence_after();
        if (kTwo) {
          __syncwarp();   // the previous tile's reads are done
          inv_stage[ew * 32 + lane] = inv4;
          __syncwarp();
        }
#pragma unroll 1
        for (int h = kTwo ? (int)(tile_it & 1u) : 0; h < 2; h += kTwo ? 2 : 1) {
#pragma unroll 1
          for (int k = 0; k < 2; k++) {
            const int cc = chunk_col(cw, k);
            const uint32_t taddr = tmem_base + (lane_base << 16) + h * 256 + cc;
            if (p.debug == 2) {   // diagnostics: no drain
              if (k == 1) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                  if (leader) mbar_arrive_relaxed(&acc_empty[h]);
                  else arrive_leader_relaxed(&acc_empty[h]);
                }
              }
              continue;
            }
            float v[kCW];
            SJB_TMEM_LD32(taddr, v, 0);
            if (kCW == 64) SJB_TMEM_LD32(taddr + 32, v, kCW - 32);
            tc_wait_ld();
            if (k == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) {
                if (leader) mbar_arrive_relaxed(&acc_empty[h]);
                else arrive_leader_relaxed(&acc_empty[h]);
              }
            }
            if (p.debug == 1) {   // diagnostics: drain, no emission
              float m = v[0];
#pragma unroll
              for (int e = 1; e < kCW; e++) m = fmaxf(m, v[e]);
              if (m > 3.0e38f) cta_sat[0] = 1u;
              continue;
            }
            const int64_t col0 =
                kTwo ? t * kTileRows + cc : t * 2 * kTileRows + h * kTileRows + cc;
            // normalise after the GEMM: (acc * inv_i) * inv_j (inv_b is
            // padded to whole 512-row tile pairs, zero past n_b)
            const float4* ib = reinterpret_cast<const float4*>(p.inv_b + col0);
            const float4* is = inv_stage + ew * 32 + (kCW / 4) * k;
#pragma unroll
            for (int q4 = 0; q4 < kCW / 4; q4++) {
              const float4 w = kTwo ? is[q4] : __ldg(ib + q4);
              v[4 * q4 + 0] = __fmul_rn(__fmul_rn(v[4 * q4 + 0], inv_i), w.x);
              v[4 * q4 + 1] = __fmul_rn(__fmul_rn(v[4 * q4 + 1], inv_i), w.y);
              v[4 * q4 + 2] = __fmul_rn(__fmul_rn(v[4 * q4 + 2], inv_i), w.z);
              v[4 * q4 + 3] = __fmul_rn(__fmul_rn(v[4 * q4 + 3], inv_i), w.w);
            }
            if (p.debug == 3) {   // diagnostics: drain + normalise, no emission
              float m = v[0];
#pragma unroll
              for (int e = 1; e < kCW; e++) m = fmaxf(m, v[e]);
              if (m > 3.0e38f) cta_sat[0] = 1u;
              continue;
            }
            if (p.tol)
              fin += emit_row_chunk_tol<kCW>(v, row_ok, p.cutoff, p.hi_cut, (uint32_t)gi64,
                                             (uint32_t)col0, p.n_b - col0, cta_cnt, cta_sat, seg,
                                             p.seg_cap, sims, pend_cnt, pend, scr);
            else
              emit_row_chunk<kCW>(v, row_ok, p.cutoff, (uint32_t)gi64, (uint32_t)col0,
                                  p.n_b - col0, cta_cnt, cta_sat, seg, p.seg_cap);
          }
        }
      }
      if (fin) atomicAdd(p.rowcount + gi64, fin);
    }
    if (toff != nullptr) {
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
      if (ew == 0 && lane == 0) toff[item_k] = *(volatile uint32_t*)cta_cnt;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();   // no peer MMA or arrive targets an exited CTA
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, 512);
  }
  if (threadIdx.x == 0) {
    p.cta_count[blockIdx.x] = *cta_sat ? ~0ull >> 1 : (unsigned long long)*cta_cnt;
    if (p.tol) p.pend_count[blockIdx.x] = *pend_cnt;
  }
}

}  // namespace wide2
}  // namespace sjb
