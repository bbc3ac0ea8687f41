// sjb_join_ts.cu -- the d <= 128 threshold filter with the R block in tensor
// memory (opt-in, SJB_FILTER=ts; measured against sjb_join.cu's SS-mode
// kernel, which stays the default: cfg2 16.8 vs 16.45 ms sustained, and the
// same 14.65 ms with the epilogue disabled -- the tensor pipe there is bound
// by the board power cap, not by shared-memory bandwidth).
//
// Same job and output as join_filter_kernel (sjb_join.cu): the fused
// R.S^T filter replacing tile_similarity + threshold_scan
// (linalg.py:116-153 -> sj_tile_dot / sj_scan_count / sj_scan_fill,
// _kernelcore.c:273-323), candidates packed into per-CTA segments and
// re-decided in canonical fp32 by the recheck warps.  What changes is where
// the operands live:
//
//   * The 256-row R block is copied once per work item from its shared
//     memory image into tensor memory (tcgen05.cp.128x256b, 7 per M=128
//     half at d = 100) and every UMMA reads A from TMEM ("TS" form).  Shared
//     memory then only feeds B: 4 KB per 128x128x16 MMA (64 B/cycle) instead
//     of 12 KB per 128x256x16 MMA (96 B/cycle) -- with the 31 B/cycle of S
//     tile TMA writes the SS kernel sits near the ~128 B/cycle shared-memory
//     limit (the hypothesis this kernel tested; see the header note).
//   * With A taking 112 TMEM columns, the accumulators are three 128-column
//     stages (N = 128): an S tile is 4 stage uses (2 R halves x 2 S halves)
//     and the epilogue has two stage-times of slack before the MMA waits,
//     which absorbs the emission of hit chunks.
//
//   warp 0 ln 0  S producer (1-D bulk copies of pre-tiled fp16 S tiles, ring)
//   warp 0 ln 1  R-block producer (one shared-memory image, freed once copied)
//   warp 1       TMEM allocator + MMA issuer (elect.sync, warp-uniform)
//   warps 2..17  epilogue: two groups of 8 alternating stage uses; warp
//                (q, c) of a group loads TMEM lanes 32q.. x 64 columns 64c..
//                (one tcgen05.ld.x64), releases the stage, then pre-filters
//                and emits -- group g always sees S half g of each tile
//   warps 18..19 canonical recheck (sj_dot_seq order), as in sjb_join.cu
#include "sjb_common.cuh"

namespace sjb {
namespace ts {

constexpr int kEpiWarps = 16;
constexpr int kRecheckWarps = 2;
constexpr int kThreads = 32 * (2 + kEpiWarps + kRecheckWarps);
constexpr int kStages = 3;        // accumulator stages of 128 fp32 columns
constexpr int kN = 128;           // UMMA N
constexpr uint32_t kAcol = kStages * kN;  // first TMEM column of the R block

struct SmemLayout {
  uint32_t tile_bytes;
  uint32_t off_b, off_bar, total;
};

__host__ __device__ inline SmemLayout smem_layout(int kpad, int stages) {
  SmemLayout L;
  L.tile_bytes = (uint32_t)kTileRows * kpad * 2;
  L.off_b = L.tile_bytes;  // one R-block image at 0
  L.off_bar = L.off_b + stages * L.tile_bytes;
  // a_full a_empty mma_done acc_full[3] acc_empty[3] b_full[S] b_empty[S]
  // + tmem slot, candidate counter, wrap flag, finished-epilogue-warp count
  L.total = L.off_bar + (9 + 2 * stages) * 8 + 16 + 16;
  return L;
}

__device__ __forceinline__ void tc_cp_128x256b_elect(uint32_t taddr, uint64_t sdesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(taddr),
      "l"(sdesc)
      : "memory");
}
__device__ __forceinline__ void tc_mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem,
                                                uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int KSTEPS>
__global__ void __launch_bounds__(kThreads, 1) filter_kernel(const JoinParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const SmemLayout L = smem_layout(p.kpad, p.stages);
  uint8_t* a_buf = smem;
  uint8_t* b_buf = smem + L.off_b;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 1;
  uint64_t* mma_done = bars + 2;
  uint64_t* acc_full = bars + 3;
  uint64_t* acc_empty = bars + 6;
  uint64_t* b_full = bars + 9;
  uint64_t* b_empty = bars + 9 + p.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9 + 2 * p.stages);
  uint32_t* cta_cnt = reinterpret_cast<uint32_t*>(bars + 9 + 2 * p.stages + 2);
  uint32_t* cta_sat = cta_cnt + 1;
  uint32_t* epi_done = cta_cnt + 2;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    mbar_init(mma_done, 1);
    for (int i = 0; i < kStages; i++) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kEpiWarps / 2);
    }
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    init_segment_count(p.cta_count, p.append != 0, cta_cnt, cta_sat);
    *epi_done = 0u;
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t n_items = p.n_items;
  const int nb = p.n_ablk;
  const uint32_t tile_bytes = L.tile_bytes;
  const uint32_t tile_elems = tile_bytes / 2;

  if (warp == 0 && lane == 1) {
    // ------------------------------------------------- R-block producer
    const uint64_t pol_a = policy_evict_last();
    int64_t it = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, it++) {
      const int64_t rb = item % nb;
      mbar_wait(a_empty, (uint32_t)(it & 1) ^ 1u);
      mbar_arrive_expect_tx(a_full, tile_bytes);
      bulk_g2s(a_buf, p.a16 + (size_t)rb * tile_elems, tile_bytes, a_full, pol_a);
    }
  } else if (warp == 0) {
    if (lane == 0) {
      // -------------------------------------------------------- S producer
      const uint64_t pol_b = policy_evict_normal();
      int bstage = 0;
      uint32_t bphase = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int64_t sc = item / nb;
        const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
        for (int64_t t = t0; t < t1; t++) {
          mbar_wait(&b_empty[bstage], bphase ^ 1u);
          mbar_arrive_expect_tx(&b_full[bstage], tile_bytes);
          bulk_g2s(b_buf + (size_t)bstage * tile_bytes, p.b16 + (size_t)t * tile_elems,
                   tile_bytes, &b_full[bstage], pol_b);
          if (++bstage == p.stages) {
            bstage = 0;
            bphase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------- MMA issuer
    const uint32_t idesc = umma_idesc_f16_f32(128, kN, true);
    const uint32_t lbo = kTileRows * 16;  // 256-row operand: distance between k-groups
    const uint32_t sbo = 128;             // distance between 8-row core-matrix groups
    const uint64_t kstep = (2 * lbo) >> 4;        // one k-step = 2 k-groups
    const uint64_t half_step = (128 * 16) >> 4;   // 128 rows further
    const uint64_t a_desc = umma_desc_kmajor_noswz(smem_u32(a_buf), lbo, sbo);
    const uint64_t b_desc_base = umma_desc_kmajor_noswz(smem_u32(b_buf), lbo, sbo);
    const uint64_t tile_step = tile_bytes >> 4;
    const uint32_t a_tm = tmem_base + kAcol;
    int bstage = 0, s = 0;
    uint32_t bphase = 0, sph = 0;
    int64_t it = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, it++) {
      const int64_t sc = item / nb;
      mbar_wait(a_full, (uint32_t)(it & 1));
      if (it > 0) {
        // the previous item's MMAs must have read the TMEM R block
        tc_commit_elect(mma_done);
        mbar_wait(mma_done, (uint32_t)((it - 1) & 1));
      }
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int kk = 0; kk < KSTEPS; kk++)
          tc_cp_128x256b_elect(a_tm + (h * KSTEPS + kk) * 8, a_desc + h * half_step + kk * kstep);
      tc_commit_elect(a_empty);   // the shared-memory image is free once copied
      const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
      const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
      for (int64_t t = t0; t < t1; t++) {
        mbar_wait(&b_full[bstage], bphase);
        const uint64_t bd = b_desc_base + (uint64_t)bstage * tile_step;
#pragma unroll
        for (int h = 0; h < 2; h++) {
#pragma unroll
          for (int n = 0; n < 2; n++) {
            mbar_wait(&acc_empty[s], sph ^ 1u);
            tc_fence_after();
            const uint32_t d = tmem_base + s * kN;
            const uint32_t ah = a_tm + h * KSTEPS * 8;
            const uint64_t bn = bd + n * half_step;
#pragma unroll
            for (int kk = 0; kk < KSTEPS; kk++)
              tc_mma_ts_elect(d, ah + kk * 8, bn + kk * kstep, idesc, kk > 0 ? 1u : 0u);
            tc_commit_elect(&acc_full[s]);
            if (++s == kStages) {
              s = 0;
              sph ^= 1u;
            }
          }
        }
        tc_commit_elect(&b_empty[bstage]);
        if (++bstage == p.stages) {
          bstage = 0;
          bphase ^= 1u;
        }
      }
    }
  } else if (warp >= 2 + kEpiWarps) {
    // ------------------------------------------------------ recheck warps
    const int rw = warp - 2 - kEpiWarps;
    const uint64_t seg_cap = p.seg_cap;
    const uint64_t* seg = p.cand + (uint64_t)blockIdx.x * seg_cap;
    uint32_t* sims = p.sims_bits + (uint64_t)blockIdx.x * seg_cap;
    if (p.debug_mode != 5 && !p.defer)  // (diagnostics: 5 = emit, no recheck, results invalid)
      recheck_loop(seg, sims, seg_cap, (volatile uint32_t*)cta_cnt, (volatile uint32_t*)epi_done,
                   (uint32_t)kEpiWarps, rw, kRecheckWarps,
                   p.l32, p.r32, p.dim, p.theta, p.rowcount,
                   p.append ? (uint64_t)p.cta_count[blockIdx.x] : 0ull);
  } else {
    // ---------------------------------------------------------- epilogue
    // Stage uses are numbered u = 0, 1, 2, ... in MMA order (per S tile:
    // (R half 0, S half 0), (0, 1), (1, 0), (1, 1)); use u lives in stage
    // u % 3 with phase (u / 3) & 1 and is drained by group u & 1, so group g
    // always drains S half g and alternates R halves.
    const int ew = warp - 2;
    const int grp = ew >> 3;
    const int cq = (ew >> 2) & 1;     // 64-column half of the 128-column stage
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const uint32_t lane_base = (uint32_t)q * 32;
    uint64_t* seg = p.cand + (uint64_t)blockIdx.x * p.seg_cap;
    const uint64_t seg_cap = p.seg_cap;
    const uint32_t tbase = tmem_base + (lane_base << 16) + (uint32_t)cq * 64;
    const bool no_drain = p.debug_mode == 2 || p.debug_mode >= 16;   // diagnostics
    const bool no_emit = p.debug_mode == 1;
    const bool per_row = p.row_err != nullptr;
    int s = grp;
    uint32_t sph = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t rb = item % nb, sc = item / nb;
      const int t0 = p.tile_begin + (int)sc * p.tiles_per_chunk;
      const int t1 = mn<int>(t0 + p.tiles_per_chunk, p.n_btiles);
      // per-row band: cutoff = max(cutoff, theta - slack - (1+1e-6)(ex + ey)
      // - ex*ey) = max(cutoff, cA - cB*ey); the 2e-6 in `slack` covers the
      // fp32 evaluation of either form
      uint32_t gi[2];
      bool rok[2];
      float cA[2], cB[2];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t g64 = rb * kTileRows + h * 128 + lane_base + lane;
        gi[h] = (uint32_t)g64;
        rok[h] = g64 < p.n_a && !no_emit;
        const float ex = load_err(p.row_err, g64, p.n_a);
        cA[h] = per_row ? p.theta - p.slack - 1.000001f * ex : p.cutoff;
        cB[h] = per_row ? 1.000001f + ex : 0.0f;
      }
      for (int t = t0; t < t1; t++) {
        // issued before the accumulator wait: its latency hides behind it
        const float ey = per_row ? __ldg(p.tile_err + t) : 0.0f;
        const uint32_t j0 = (uint32_t)t * kTileRows + grp * kN + cq * 64;
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int su = s;
          mbar_wait(&acc_full[su], sph);
          tc_fence_after();
          if (s + 2 >= kStages) { s += 2 - kStages; sph ^= 1u; } else { s += 2; }
          if (no_drain) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[su]);
            continue;
          }
          float v[64];
          SJB_TMEM_LD64(tbase + su * kN, v);
          tc_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_relaxed(&acc_empty[su]);
          const float cutoff = fmaxf(p.cutoff, fmaf(-cB[h], ey, cA[h]));
          float g[8];
#pragma unroll
          for (int k = 0; k < 8; k++) {
            const float* x = v + 8 * k;
            g[k] = fmax3(fmax3(x[0], x[1], x[2]), fmax3(x[3], x[4], x[5]), fmaxf(x[6], x[7]));
          }
          const float m =
              fmax3(fmax3(g[0], g[1], g[2]), fmax3(g[3], g[4], g[5]), fmaxf(g[6], g[7]));
          const bool hit = rok[h] && (m >= cutoff);
          if (__any_sync(0xffffffffu, hit)) {
            // hit lanes: 64-bit mask of the columns >= cutoff (inside groups
            // whose maximum hit); one shared atomic per warp reserves slots
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
              const int64_t col_lim = p.n_b - (int64_t)j0;  // columns >= col_lim: padding
              if (col_lim < 64) {
                const int cl = (int)mx<int64_t>(col_lim, 0);
                mk0 &= cl >= 32 ? ~0u : ((1u << cl) - 1u);
                mk1 &= cl <= 32 ? 0u : ((1u << (cl - 32)) - 1u);
              }
            }
            const uint32_t cnt = __popc(mk0) + __popc(mk1);
            uint64_t pos;
            if (__popc(__ballot_sync(0xffffffffu, cnt != 0)) <= 1) {
              uint32_t base = 0;
              if (cnt) {
                base = atomicAdd(cta_cnt, cnt);
                if (base + cnt < base) *cta_sat = 1u;
              }
              pos = base;
            } else {
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
              pos = (uint64_t)base + (incl - cnt);
            }
            uint32_t w = mk0;
            while (w) {
              const int b = __ffs(w) - 1;
              w &= w - 1;
              if (pos < seg_cap) seg[pos] = pack_pair(gi[h], j0 + b);
              pos++;
            }
            w = mk1;
            while (w) {
              const int b = __ffs(w) - 1;
              w &= w - 1;
              if (pos < seg_cap) seg[pos] = pack_pair(gi[h], j0 + 32 + b);
              pos++;
            }
          }
        }
      }
    }
    // publish "this warp reserved its last slots" to the recheck warps
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
  // saturated counters report an impossible count so the host raises
  if (threadIdx.x == 0)
    p.cta_count[blockIdx.x] = *cta_sat ? ~0ull >> 1 : (unsigned long long)*cta_cnt;
}

}  // namespace ts
}  // namespace sjb
