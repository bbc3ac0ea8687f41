// sjb_join.cu -- the fused R.S^T threshold filter (the hot path).
//
// Replaces the reference's tile_similarity + threshold_scan pair
// (linalg.py:116-153 -> sj_tile_dot _kernelcore.c:300-323 + sj_scan_count/fill
// :327-350) with one persistent, warp-specialised tcgen05 kernel that never
// materialises the similarity matrix:
//
//   warp 0      producer: 1-D bulk copies (TMA, cp.async.bulk) of pre-tiled
//               bf16 operand tiles into shared memory (mbarrier ring)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..9  epilogue: tcgen05.ld of the fp32 accumulators, 3-input max
//               pre-filter against (theta - band), candidate emission
//
// Work item = (R block of 256 rows, S chunk of `tiles_per_chunk` 128-row
// tiles).  The R block (two M=128 UMMA operands) stays resident in shared
// memory (double-buffered across items) while the chunk's S tiles stream
// through a multi-stage ring; each S tile is one 256x128 output tile =
// 2 x (kpad/16) UMMA_128x128x16 instructions into a TMEM accumulator stage
// (2 stages x 256 columns = all 512 TMEM columns).  Items are ordered
// S-chunk-major so the CTAs resident at any moment share the same S chunk
// in L2.
//
// Output: candidate pairs (i, j) with bf16 approx >= cutoff, packed as
// u64 (i << 32 | j) into per-CTA segments of `cand` (seg_cap each), counted in
// a shared-memory counter and published in cta_count[blockIdx.x].  A CTA
// whose segment overflows keeps counting, so the host can retry with the
// exact capacity (the schedule is static, so per-CTA counts are
// reproducible).  Every candidate is re-decided in canonical fp32 by
// sjb_post.cu's recheck kernel.
#include "sjb_common.cuh"

namespace sjb {

constexpr int kJoinThreads = 320;
constexpr int kEpiWarps = 8;
constexpr int kBM = 256;  // resident R rows per item (two UMMA M=128 halves)
constexpr int kBN = 128;  // S rows per stage == UMMA N

struct JoinParams {
  const __nv_bfloat16* a16;  // R operand image, 2*n_ablk tiles
  const __nv_bfloat16* b16;  // S operand image, n_btiles tiles
  int64_t n_a, n_b;          // valid rows
  int kpad;                  // padded K (multiple of 16, <= 128)
  int n_ablk;                // ceil(n_a / 256)
  int n_btiles;              // ceil(n_b / 128)
  int tiles_per_chunk;
  int64_t n_items;
  int stages;
  float cutoff;
  uint64_t* cand;
  uint64_t seg_cap;
  unsigned long long* cta_count;
  int debug_mode;  // diagnostics: 0 normal, 1 no emission, 2 no TMEM drain, 3 spin waits
};

struct JoinSmemLayout {
  uint32_t a_bytes, b_bytes;  // per buffer
  uint32_t off_a0, off_a1, off_b, off_bar, total;
};

__host__ __device__ inline JoinSmemLayout join_smem_layout(int kpad, int stages) {
  JoinSmemLayout L;
  L.a_bytes = (uint32_t)kBM * kpad * 2;
  L.b_bytes = (uint32_t)kBN * kpad * 2;
  L.off_a0 = 0;
  L.off_a1 = L.a_bytes;
  L.off_b = 2 * L.a_bytes;
  L.off_bar = L.off_b + stages * L.b_bytes;
  // a_full[2] a_empty[2] acc_full[2] acc_empty[2] b_full[S] b_empty[S] + tmem slot + counter
  L.total = L.off_bar + (8 + 2 * stages) * 8 + 16 + 16;
  return L;
}

// KSTEPS = kpad / 16 UMMA k-steps per output tile (compile time so the issue
// loop is straight-line: each tcgen05.mma costs one descriptor add).
template <int KSTEPS>
__global__ void __launch_bounds__(kJoinThreads, 1) join_filter_kernel(const JoinParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const JoinSmemLayout L = join_smem_layout(p.kpad, p.stages);
  uint8_t* a_buf[2] = {smem + L.off_a0, smem + L.off_a1};
  uint8_t* b_buf = smem + L.off_b;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 2;
  uint64_t* acc_full = bars + 4;
  uint64_t* acc_empty = bars + 6;
  uint64_t* b_full = bars + 8;
  uint64_t* b_empty = bars + 8 + p.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * p.stages);
  // 32-bit shared counter (native ATOMS.ADD); cta_sat latches a wrap-around
  // so the host reports it instead of trusting a truncated count.
  uint32_t* cta_cnt = reinterpret_cast<uint32_t*>(bars + 8 + 2 * p.stages + 2);
  uint32_t* cta_sat = cta_cnt + 1;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; i++) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kEpiWarps);
    }
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    *cta_cnt = 0u;
    *cta_sat = 0u;
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t n_items = p.n_items;
  const int nb = p.n_ablk;
  const uint32_t tile_elems = (uint32_t)kBN * p.kpad;  // elements per 128-row tile
  const uint32_t tile_bytes = tile_elems * 2;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer
      const uint64_t pol_a = policy_evict_last();
      const uint64_t pol_b = policy_evict_normal();
      int bstage = 0;
      uint32_t bphase = 0;
      int64_t it = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, it++) {
        const int64_t rb = item % nb, sc = item / nb;
        const int ab = (int)(it & 1);
        mbar_wait(&a_empty[ab], (uint32_t)((it >> 1) & 1) ^ 1u);
        mbar_arrive_expect_tx(&a_full[ab], 2 * tile_bytes);
        const __nv_bfloat16* asrc = p.a16 + (size_t)(2 * rb) * tile_elems;
        bulk_g2s(a_buf[ab], asrc, tile_bytes, &a_full[ab], pol_a);
        bulk_g2s(a_buf[ab] + tile_bytes, asrc + tile_elems, tile_bytes, &a_full[ab], pol_a);
        const int64_t t0 = sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
        for (int64_t t = t0; t < t1; t++) {
          mbar_wait(&b_empty[bstage], bphase ^ 1u);
          if (p.debug_mode == 17 && it > 0) {
            mbar_arrive(&b_full[bstage]);  // diagnostics: no B traffic after the first item
          } else {
            const int64_t tl = p.debug_mode == 16 ? (t & 7) : t;  // diagnostics: hot B set
            mbar_arrive_expect_tx(&b_full[bstage], tile_bytes);
            bulk_g2s(b_buf + (size_t)bstage * L.b_bytes, p.b16 + (size_t)tl * tile_elems,
                     tile_bytes, &b_full[bstage], pol_b);
          }
          if (++bstage == p.stages) {
            bstage = 0;
            bphase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------- MMA issuer
      const uint32_t idesc = umma_idesc_bf16_f32(128, kBN);
      const uint32_t lbo = kBN * 16;  // 128-row operand: distance between k-groups
      const uint32_t sbo = 128;       // distance between 8-row core-matrix groups
      // descriptor of each buffer at k-step 0; a k-step advances the start
      // address by 2 k-groups = 2 * lbo bytes (encoded >> 4)
      const uint64_t kstep = (2 * lbo) >> 4;
      const uint64_t a_desc0[2] = {umma_desc_kmajor_noswz(smem_u32(a_buf[0]), lbo, sbo),
                                   umma_desc_kmajor_noswz(smem_u32(a_buf[1]), lbo, sbo)};
      const uint64_t b_desc_base = umma_desc_kmajor_noswz(smem_u32(b_buf), lbo, sbo);
      const uint64_t half_step = tile_bytes >> 4;       // second A half
      const uint64_t stage_step = L.b_bytes >> 4;
      int bstage = 0;
      uint32_t bphase = 0;
      uint32_t acc_it = 0;
      int64_t it = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, it++) {
        const int64_t sc = item / nb;
        const int ab = (int)(it & 1);
        mbar_wait(&a_full[ab], (uint32_t)((it >> 1) & 1));
        tc_fence_after();
        const uint64_t ad = a_desc0[ab];
        const int64_t t0 = sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
        for (int64_t t = t0; t < t1; t++) {
          const uint32_t as = acc_it & 1u;
          mbar_wait(&acc_empty[as], ((acc_it >> 1) & 1u) ^ 1u);
          mbar_wait(&b_full[bstage], bphase);
          tc_fence_after();
          const uint64_t bd = b_desc_base + (uint64_t)bstage * stage_step;
          const uint32_t d0 = tmem_base + as * 256;
#pragma unroll
          for (int kk = 0; kk < KSTEPS; kk++)
            tc_mma_bf16(d0, ad + kk * kstep, bd + kk * kstep, idesc, kk > 0 ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < KSTEPS; kk++)
            tc_mma_bf16(d0 + 128, ad + half_step + kk * kstep, bd + kk * kstep, idesc,
                        kk > 0 ? 1u : 0u);
          tc_commit(&b_empty[bstage]);
          tc_commit(&acc_full[as]);
          if (++bstage == p.stages) {
            bstage = 0;
            bphase ^= 1u;
          }
          acc_it++;
        }
        tc_commit(&a_empty[ab]);
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    const int ew = warp - 2;
    const int h = ew >> 2;            // accumulator half (R rows 0-127 / 128-255)
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const uint32_t lane_base = (uint32_t)q * 32;
    const float cutoff = p.cutoff;
    uint64_t* seg = p.cand + (uint64_t)blockIdx.x * p.seg_cap;
    const uint64_t seg_cap = p.seg_cap;
    uint32_t acc_it = 0;
    uint32_t dbg_acc = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t rb = item % nb, sc = item / nb;
      const int64_t gi64 = rb * kBM + h * 128 + lane_base + lane;
      const bool row_ok = gi64 < p.n_a;
      const uint32_t gi = (uint32_t)gi64;
      const int64_t t0 = sc * p.tiles_per_chunk;
      const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
      for (int64_t t = t0; t < t1; t++) {
        const uint32_t as = acc_it & 1u;
        mbar_wait(&acc_full[as], (acc_it >> 1) & 1u);
        tc_fence_after();
        if (p.debug_mode == 2 || p.debug_mode >= 16) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[as]);
          acc_it++;
          continue;
        }
        float v[128];
        const uint32_t taddr = tmem_base + (lane_base << 16) + as * 256 + h * 128;
        SJB_TMEM_LD32(taddr + 0, v, 0);
        SJB_TMEM_LD32(taddr + 32, v, 32);
        SJB_TMEM_LD32(taddr + 64, v, 64);
        SJB_TMEM_LD32(taddr + 96, v, 96);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (p.debug_mode == 5) mbar_arrive(&acc_empty[as]);
          else mbar_arrive_relaxed(&acc_empty[as]);
        }
        acc_it++;

        // group maxima over 8 columns, then the tile maximum
        float g[16];
#pragma unroll
        for (int k = 0; k < 16; k++) {
          const float* x = v + 8 * k;
          g[k] = fmax3(fmax3(x[0], x[1], x[2]), fmax3(x[3], x[4], x[5]), fmaxf(x[6], x[7]));
        }
        float m = fmax3(fmax3(g[0], g[1], g[2]), fmax3(g[3], g[4], g[5]),
                        fmax3(g[6], g[7], g[8]));
        m = fmax3(m, fmax3(g[9], g[10], g[11]), fmax3(g[12], g[13], fmaxf(g[14], g[15])));
        const bool hit = row_ok && (m >= cutoff) && p.debug_mode != 1;
        if (__any_sync(0xffffffffu, hit)) {
          // Slow path (warp-uniform): each hit thread builds a 128-bit mask of
          // its columns >= cutoff (only inside groups whose maximum hit), then
          // one warp scan + one shared atomic reserve the warp's slots and each
          // thread writes its pairs -- no collectives per candidate.
          uint32_t mk0 = 0, mk1 = 0, mk2 = 0, mk3 = 0;
          if (hit) {
#pragma unroll
            for (int k = 0; k < 16; k++) {
              if (g[k] >= cutoff) {
                uint32_t b = 0;
#pragma unroll
                for (int e = 0; e < 8; e++) b |= (v[8 * k + e] >= cutoff ? 1u : 0u) << e;
                const uint32_t sh = b << (8 * (k & 3));
                if ((k >> 2) == 0) mk0 |= sh;
                else if ((k >> 2) == 1) mk1 |= sh;
                else if ((k >> 2) == 2) mk2 |= sh;
                else mk3 |= sh;
              }
            }
            const int64_t col_lim = p.n_b - t * kBN;  // columns >= col_lim are padding
            if (col_lim < 128) {
              const int cl = (int)col_lim;
              mk0 &= cl >= 32 ? ~0u : ((1u << cl) - 1u);
              mk1 &= cl >= 64 ? ~0u : (cl <= 32 ? 0u : ((1u << (cl - 32)) - 1u));
              mk2 &= cl >= 96 ? ~0u : (cl <= 64 ? 0u : ((1u << (cl - 64)) - 1u));
              mk3 &= cl <= 96 ? 0u : ((1u << (cl - 96)) - 1u);
            }
          }
          const uint32_t cnt = __popc(mk0) + __popc(mk1) + __popc(mk2) + __popc(mk3);
          if (p.debug_mode == 4) {  // diagnostics: masks only
            dbg_acc += cnt;
            continue;
          }
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
          const uint32_t j0 = (uint32_t)(t * kBN);
          const uint32_t mks[4] = {mk0, mk1, mk2, mk3};
#pragma unroll
          for (int q2 = 0; q2 < 4; q2++) {
            uint32_t w = mks[q2];
            while (w) {
              const int b = __ffs(w) - 1;
              w &= w - 1;
              if (pos < seg_cap && p.debug_mode != 3) seg[pos] = pack_pair(gi, j0 + 32 * q2 + b);
              pos++;
            }
          }
        }
      }
    }
    if (p.debug_mode == 4 && dbg_acc == 0xFFFFFFFFu) p.cand[0] = dbg_acc;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
  // saturated counters report an impossible count so the host raises
  if (threadIdx.x == 0) p.cta_count[blockIdx.x] = *cta_sat ? ~0ull >> 1 : (unsigned long long)*cta_cnt;
}

}  // namespace sjb
