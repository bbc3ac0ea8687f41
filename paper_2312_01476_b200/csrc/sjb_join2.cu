// sjb_join2.cu -- the fused threshold filter on CTA PAIRS (cta_group::2).
//
// Same contract as sjb_join.cu (candidates with fp16 approx >= cutoff into
// per-CTA segments, fused canonical recheck), organised for a 2-SM pair:
//
//   * Each CTA keeps its own 256-row R block resident (two M=128 halves);
//     the pair block is 512 R rows.  One UMMA_256x128x16 (cta_group::2,
//     issued by the leader CTA) multiplies the h-half of BOTH CTAs' blocks
//     (256 rows) by a 128-row S tile whose rows 0-63 sit in the leader's
//     shared memory and 64-127 in the peer's.
//   * Each CTA's TMEM receives its own 128 rows x 128 columns per stage, so
//     the 512 columns hold FOUR accumulator stages (1-CTA N=256 held two):
//     the tensor core can run three stages ahead of the epilogue.
//   * Shared-memory operand reads are 96 B/cycle per SM (A 4 KB + B 2 KB per
//     64-cycle MMA) and the S tile is fetched once per 512 R rows (half the
//     L2->SM traffic of the 1-CTA kernel).
//
// Warp roles per CTA (20 warps):
//   warp 0 lane 0  S producer: one 2-SM tensor TMA per stage (this CTA's
//                  64-row half of the 128-row S tile) -> B ring
//   warp 0 lane 1  R-block producer
//   warp 1         TMEM allocation (cta_group::2); lane 0 of the leader CTA
//                  issues every MMA of the pair
//   warps 2..17    epilogue, two groups of 8 taking alternate stages; a warp
//                  drains 32 lanes x 64 columns of every other stage, so it
//                  has two stage-times (~900 cycles) per stage it owns, and
//                  the four TMEM stages absorb emission-heavy stages
//   warps 18..19   canonical recheck of this CTA's candidates
//
// Operand delivery: 3-D TMA tensor copies with .cta_group::2.  The operand
// image (256-row tiles, [k-group][row][8 elements]) is described as a tensor
// (8 elements, 256 rows, k-groups x tiles); a box {8, 64 | 256, k-groups}
// lands exactly the [k-group][rows][8] shared-memory layout the UMMA
// descriptor reads, in ONE instruction, and its transaction bytes complete on
// the LEADER's barrier directly (no forwarding).  The leader posts
// expect_tx for both halves.  MMA commits are multicast to both CTAs'
// b_empty / a_empty / acc_full; the leader's acc_empty counts the epilogue
// warps of both CTAs (peer warps arrive remotely, relaxed).
#include <cuda.h>

#include "sjb_common.cuh"

#ifndef SJB_PROFILE
#define SJB_PROFILE 0
#endif

namespace sjb {

namespace pair {

// 16 epilogue warps in two stage-alternating groups of 8, each warp 32 lanes x
// 64 columns (64 values amortise the per-stage fixed costs; 16 warps x 32
// columns of EVERY stage was issue-bound).
#ifndef SJB_PAIR_N
#define SJB_PAIR_N 128
#endif
constexpr int kEpiWarps = 16;
constexpr int kRecheckWarps = 2;
constexpr int kThreads = 32 * (2 + kEpiWarps + kRecheckWarps);
// Pair N = S rows per stage.  N = 256: per SM an UMMA reads 128 A rows + 128
// B rows (64 B/cycle of SMEM, the 1-CTA N=256 kernel reads 96), two TMEM
// stages, all 16 epilogue warps on every stage.  N = 128: four TMEM stages,
// two stage-alternating groups of 8 epilogue warps.
constexpr int kUmmaN = SJB_PAIR_N;
constexpr int kHalfN = kUmmaN / 2;       // S rows per CTA per stage
constexpr int kAccStages = 512 / kUmmaN;
constexpr int kEpiGroup = kUmmaN / 16;   // warps per stage: 4 lane quarters x N/64 column chunks
constexpr int kGroups = kEpiWarps / kEpiGroup;
static_assert(kUmmaN == 128 || kUmmaN == 256, "pair N");
constexpr int kARows = kTileRows;  // 256 resident R rows per CTA
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clears the CTA-rank bit of a pair smem address

struct alignas(64) Params {
  CUtensorMap tmap_a;        // R image as (8, 256, kgroups * tiles), box {8, 256, kgroups}
  CUtensorMap tmap_b;        // S image, box {8, 64, kgroups}
  const op16_t* a16;  // R operand image (256-row tiles)
  const op16_t* b16;  // S operand image (256-row tiles)
  int64_t n_a, n_b;
  int kpad;
  int n_ablk;        // ceil(n_a / 512): pair R blocks
  int n_btiles;      // ceil(n_b / 128): pair S tiles
  int tiles_per_chunk;
  int tile_begin;    // first pair S tile of this launch
  int append;        // 1: continue the segments of an earlier launch
  int64_t n_items;
  int stages;
  float cutoff;
  const float* row_err;   // per-row band (or nullptr: uniform cutoff)
  const float* tile_err;
  float slack;
  uint64_t* cand;
  uint64_t seg_cap;
  unsigned long long* cta_count;
  const float* l32;
  const float* r32;
  int dim;
  float theta;
  uint32_t* sims_bits;
  uint32_t* rowcount;
  int debug_mode;
};

struct Layout {
  uint32_t a_bytes, b_bytes, off_a, off_b, off_bar, total;
};

__host__ __device__ inline Layout layout(int kpad, int stages) {
  Layout L;
  L.a_bytes = (uint32_t)kARows * kpad * 2;
  L.b_bytes = (uint32_t)kHalfN * kpad * 2;
  L.off_a = 0;
  L.off_b = 2 * L.a_bytes;
  L.off_bar = L.off_b + stages * L.b_bytes;
  // a_full[2] a_empty[2] a_peer[2] acc_full[4] acc_empty[4] b_full[S] b_empty[S] b_peer[S]
  // + tmem slot + counters
  L.total = L.off_bar + (14 + 3 * stages) * 8 + 16 + 16;
  return L;
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// Arrive on the barrier at the same offset in the leader CTA (release at
// cluster scope so the peer's completed copies are ordered before it).
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  const uint32_t a = smem_u32(bar) & kPeerMask;
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
// Relaxed remote arrive: used for the accumulator hand-off, which publishes
// no memory (the TMEM reads are complete after tcgen05.wait::ld), so the
// epilogue's outstanding candidate stores never delay the MMA.
__device__ __forceinline__ void arrive_leader_relaxed(uint64_t* bar) {
  const uint32_t a = smem_u32(bar) & kPeerMask;
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
// 3-D tensor TMA into this CTA's shared memory, completing on the leader's
// barrier (address with the CTA-rank bit cleared).
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
// Issued by a whole warp in warp-uniform control flow; one elected lane
// executes the instruction.  Keeping the issuing code uniform lets the
// compiler hold descriptors in uniform registers: a divergent single-lane
// issue cost ~15 instructions (ELECT loop + R2UR moves) per MMA, more than
// the 64-cycle UMMA_256x128x16 itself.
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
// Commit the pair's prior MMAs to the barrier at this offset in both CTAs
// (warp-uniform, elected lane).
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

template <int KSTEPS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    filter_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const Layout L = layout(p.kpad, p.stages);
  uint8_t* a_buf = smem + L.off_a;
  uint8_t* b_buf = smem + L.off_b;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* a_full = bars + 0;     // leader: local tx + peer forward
  uint64_t* a_empty = bars + 2;    // both: MMA commit (multicast)
  uint64_t* a_local = bars + 4;    // peer: own copy landed
  uint64_t* acc_full = bars + 6;   // both: MMA commit (multicast)
  uint64_t* acc_empty = bars + 10; // leader: epilogue warps of both CTAs
  uint64_t* b_full = bars + 14;
  uint64_t* b_empty = bars + 14 + p.stages;
  uint64_t* b_local = bars + 14 + 2 * p.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14 + 3 * p.stages);
  uint32_t* cta_cnt = reinterpret_cast<uint32_t*>(bars + 14 + 3 * p.stages + 2);
  uint32_t* cta_sat = cta_cnt + 1;
  uint32_t* epi_done = cta_cnt + 2;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair_id = blockIdx.x >> 1;
  const int n_pairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; i++) {
      mbar_init(&a_full[i], 1);   // leader: expect_tx for both CTAs' tiles
      mbar_init(&a_empty[i], 1);
      mbar_init(&a_local[i], 1);
    }
    for (int i = 0; i < kAccStages; i++) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 2 * kEpiGroup);
    }
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
      mbar_init(&b_local[s], 1);
    }
    init_segment_count(p.cta_count, p.append != 0, cta_cnt, cta_sat);
    *epi_done = 0u;
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t n_items = p.n_items;
  const int nb = p.n_ablk;
  const uint32_t kgroups = (uint32_t)p.kpad / 8;

  if (warp == 0 && lane == 1) {
    // ------------------------------------------------- R-block producer
    const uint64_t pol = policy_evict_last();
    int64_t it = 0;
    for (int64_t item = pair_id; item < n_items; item += n_pairs, it++) {
      const int64_t rb = item % nb;
      const int ab = (int)(it & 1);
      mbar_wait(&a_empty[ab], (uint32_t)((it >> 1) & 1) ^ 1u);
      if (leader) mbar_arrive_expect_tx(&a_full[ab], 2 * L.a_bytes);
      // this CTA's 256-row tile (2 * rb + rank) of the pair's 512-row block
      tma3d_2sm(a_buf + (size_t)ab * L.a_bytes, &p.tmap_a, 0, 0, (int)((2 * rb + rank) * kgroups),
                &a_full[ab], pol);
    }
  } else if (warp == 0 && lane == 0) {
    // -------------------------------------------------------- S producer
    const uint64_t pol = policy_evict_normal();
    int bstage = 0;
    uint32_t bphase = 0;
    for (int64_t item = pair_id; item < n_items; item += n_pairs) {
      const int64_t sc = item / nb;
      const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
      const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
      for (int64_t t = t0; t < t1; t++) {
        mbar_wait(&b_empty[bstage], bphase ^ 1u);
        // pair tile t = S rows [128t, 128t+128); this CTA owns rows
        // r0 = 128t + 64*rank: image tile r0/256, rows r0%256 .. +63
        const int64_t r0 = t * kUmmaN + rank * kHalfN;
        if (p.debug_mode == 20 && t >= p.stages) {  // diagnostics: no S traffic after the ring filled
          if (leader) mbar_arrive(&b_full[bstage]);
        } else {
          if (leader) mbar_arrive_expect_tx(&b_full[bstage], 2 * L.b_bytes);
          tma3d_2sm(b_buf + (size_t)bstage * L.b_bytes, &p.tmap_b, 0,
                    (int)(r0 % kTileRows) / 32, (int)((r0 / kTileRows) * kgroups),
                    &b_full[bstage], pol);
        }
        if (++bstage == p.stages) {
          bstage = 0;
          bphase ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // the whole warp runs the issue loop; mma2/commit2 elect one lane
      // ---------------------------------------------- MMA issuer (pair)
      const uint32_t idesc = umma_idesc_f16_f32(256, kUmmaN, true);
      const uint32_t a_lbo = kARows * 16;   // A: 256-row block, k-group stride
      const uint32_t b_lbo = kHalfN * 16;   // B: this CTA's kHalfN-row slab, k-group stride
      const uint32_t sbo = 128;
      const uint64_t a_kstep = (2 * a_lbo) >> 4, b_kstep = (2 * b_lbo) >> 4;
      const uint64_t half_step = (128 * 16) >> 4;
      const uint64_t a_base = umma_desc_kmajor_noswz(smem_u32(a_buf), a_lbo, sbo);
      const uint64_t b_base = umma_desc_kmajor_noswz(smem_u32(b_buf), b_lbo, sbo);
      const uint64_t a_buf_step = L.a_bytes >> 4, b_stage_step = L.b_bytes >> 4;
      int bstage = 0;
      uint32_t bphase = 0;
      uint32_t acc_it = 0;
      int64_t it = 0;
      const bool dbg = SJB_PROFILE && p.debug_mode == 9;
      long long w_a = 0, w_b = 0, w_e = 0, c0 = 0;
      const long long c_start = clock64();
      for (int64_t item = pair_id; item < n_items; item += n_pairs, it++) {
        const int64_t sc = item / nb;
        const int ab = (int)(it & 1);
        if (dbg) c0 = clock64();
        mbar_wait(&a_full[ab], (uint32_t)((it >> 1) & 1));
        if (dbg) w_a += clock64() - c0;
        tc_fence_after();
        const uint64_t ad = a_base + (uint64_t)ab * a_buf_step;
        const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
        for (int64_t t = t0; t < t1; t++) {
          if (dbg) c0 = clock64();
          mbar_wait(&b_full[bstage], bphase);
          if (dbg) w_b += clock64() - c0;
          tc_fence_after();
          const uint64_t bd = b_base + (uint64_t)bstage * b_stage_step;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const uint32_t as = acc_it % kAccStages;
            if (dbg) c0 = clock64();
            mbar_wait(&acc_empty[as], ((acc_it / kAccStages) & 1u) ^ 1u);
            if (dbg) w_e += clock64() - c0;
            tc_fence_after();
            const uint32_t d = tmem_base + as * kUmmaN;
            const uint64_t adh = ad + h * half_step;
#pragma unroll
            for (int kk = 0; kk < KSTEPS; kk++)
              mma2(d, adh + kk * a_kstep, bd + kk * b_kstep, idesc, kk > 0 ? 1u : 0u);
            commit2(&acc_full[as]);
            acc_it++;
          }
          commit2(&b_empty[bstage]);
          if (++bstage == p.stages) {
            bstage = 0;
            bphase ^= 1u;
          }
        }
        commit2(&a_empty[ab]);
      }
      if (dbg && blockIdx.x < 6)
        printf("[dbg] pair %d mma: total %lld  wait_a %lld  wait_b %lld  wait_acc_empty %lld  stages %d\n",
               pair_id, clock64() - c_start, w_a, w_b, w_e, p.stages);
    }
  } else if (warp >= 2 + kEpiWarps) {
    // ------------------------------------------------------ recheck warps
    const int rw = warp - 2 - kEpiWarps;
    const uint64_t seg_cap = p.seg_cap;
    const uint64_t* seg = p.cand + (uint64_t)blockIdx.x * seg_cap;
    uint32_t* sims = p.sims_bits + (uint64_t)blockIdx.x * seg_cap;
    volatile uint32_t* vcnt = cta_cnt;
    volatile uint32_t* vdone = epi_done;
    recheck_loop(seg, sims, seg_cap, vcnt, vdone, (uint32_t)kEpiWarps, rw, kRecheckWarps, p.l32,
                 p.r32, p.dim, p.theta, p.rowcount, p.append ? (uint64_t)p.cta_count[blockIdx.x] : 0ull);
  } else if (warp >= 2) {
    // ---------------------------------------------------------- epilogue
    // warp (q, c): TMEM lanes 32q..32q+31 (this CTA's R rows of the stage's
    // half) x columns 64c..64c+63 (S rows of the pair tile).  The accumulator
    // is released right after the drain; with four TMEM stages the MMA runs
    // ahead while the warp reduces and emits.
    const int ew = warp - 2;
    const int grp = ew / kEpiGroup;          // stages k with k % kGroups == grp
    const int cq = (ew % kEpiGroup) >> 2;
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)q * 32;
    uint64_t* seg = p.cand + (uint64_t)blockIdx.x * p.seg_cap;
    const uint64_t seg_cap = p.seg_cap;
    const uint32_t tcol = tmem_base + (lane_base << 16) + cq * 64;
    const bool drain = p.debug_mode != 19 && p.debug_mode != 20;

    // stage iterator over (item, tile, half) in the MMA's issue order
    struct Stage {
      int64_t item, rb, t, t1;
      int h;
      bool valid;
    };
    auto first_of = [&](int64_t item) {
      Stage s;
      s.item = item;
      s.valid = item < n_items;
      s.h = 0;
      s.rb = item % nb;
      const int64_t sc = item / nb;
      s.t = p.tile_begin + sc * p.tiles_per_chunk;
      s.t1 = mn<int64_t>(s.t + p.tiles_per_chunk, p.n_btiles);
      return s;
    };
    auto advance = [&](Stage s) {
      if (++s.h < 2) return s;
      s.h = 0;
      if (++s.t < s.t1) return s;
      return first_of(s.item + n_pairs);
    };
    auto release = [&](uint32_t as) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive_relaxed(&acc_empty[as]);
        else arrive_leader_relaxed(&acc_empty[as]);
      }
    };
    auto row_of = [&](const Stage& s) {
      return s.rb * (2 * kARows) + rank * kARows + s.h * 128 + lane_base + lane;
    };
    auto process = [&](const float* v, const Stage& s, float cutoff) {
      if (p.debug_mode == 2 || !drain) return;
      const int64_t gi64 = row_of(s);
      const bool row_ok = gi64 < p.n_a;
      float g[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const float* x = v + 8 * k;
        g[k] = fmax3(fmax3(x[0], x[1], x[2]), fmax3(x[3], x[4], x[5]), fmaxf(x[6], x[7]));
      }
      const float m = fmax3(fmax3(g[0], g[1], g[2]), fmax3(g[3], g[4], g[5]), fmaxf(g[6], g[7]));
      const bool hit = row_ok && (m >= cutoff) && p.debug_mode != 1;
      if (!__any_sync(0xffffffffu, hit)) return;
      uint32_t mk0 = 0, mk1 = 0;
      if (hit) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
          if (g[k] >= cutoff) {
            uint32_t b = 0;
#pragma unroll
            for (int e = 0; e < 8; e++) b |= (v[8 * k + e] >= cutoff ? 1u : 0u) << e;
            if (k < 4) mk0 |= b << (8 * k);
            else mk1 |= b << (8 * (k - 4));
          }
        }
        const int64_t col_lim = p.n_b - s.t * kUmmaN - cq * 64;
        if (col_lim < 64) {
          const int cl = (int)mx<int64_t>(col_lim, 0);
          mk0 &= cl >= 32 ? ~0u : ((1u << cl) - 1u);
          mk1 &= cl <= 32 ? 0u : ((1u << (cl - 32)) - 1u);
        }
      }
      const uint32_t cnt = __popc(mk0) + __popc(mk1);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
      uint32_t base = 0;
      if (lane == 31 && wtot) {
        base = atomicAdd(cta_cnt, wtot);
        if (base + wtot < base) *cta_sat = 1u;
      }
      base = __shfl_sync(0xffffffffu, base, 31);
      uint64_t pos = (uint64_t)base + (incl - cnt);
      const uint32_t gi = (uint32_t)gi64;
      const uint32_t j0 = (uint32_t)(s.t * kUmmaN + cq * 64);
      uint32_t w = mk0;
      while (w) {
        const int b = __ffs(w) - 1;
        w &= w - 1;
        if (pos < seg_cap) seg[pos] = pack_pair(gi, j0 + b);
        pos++;
      }
      w = mk1;
      while (w) {
        const int b = __ffs(w) - 1;
        w &= w - 1;
        if (pos < seg_cap) seg[pos] = pack_pair(gi, j0 + 32 + b);
        pos++;
      }
    };
    // issue the load of stage k into `v` (after its accumulator is full)
#define SJB_PAIR_LOAD(k, v)                                                  \
  do {                                                                       \
    const uint32_t as_ = (k) % kAccStages;                                   \
    mbar_wait(&acc_full[as_], ((k) / kAccStages) & 1u);                      \
    tc_fence_after();                                                        \
    if (drain) {                                                             \
      SJB_TMEM_LD32(tcol + as_ * kUmmaN, v, 0);                              \
      SJB_TMEM_LD32(tcol + as_ * kUmmaN + 32, v, 32);                        \
    }                                                                        \
  } while (0)

    float va[64];
    uint32_t k = grp;
    Stage cur = first_of(pair_id);
    for (int g = 0; g < grp; g++) cur = advance(cur);
    for (; cur.valid; k += kGroups) {
      // band terms issued before the accumulator wait (latency hidden)
      const bool per_row = p.row_err != nullptr;
      const float ex = load_err(p.row_err, row_of(cur), p.n_a);
      const float ey = per_row ? __ldg(p.tile_err + (cur.t * kUmmaN) / kTileRows) : 0.0f;
      SJB_PAIR_LOAD(k, va);
      tc_wait_ld();
      release(k % kAccStages);
      process(va, cur, per_row ? cutoff_from(p.cutoff, p.theta, p.slack, ex, ey) : p.cutoff);
      for (int g = 0; g < kGroups; g++) cur = advance(cur);
    }
#undef SJB_PAIR_LOAD
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      atomicAdd(epi_done, 1u);
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, 512);
  }
  if (threadIdx.x == 0)
    p.cta_count[blockIdx.x] = *cta_sat ? ~0ull >> 1 : (unsigned long long)*cta_cnt;
}

}  // namespace pair
}  // namespace sjb
