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
          mbar_arrive_expect_tx(&b_full[bstage], tile_bytes);
          bulk_g2s(b_buf + (size_t)bstage * L.b_bytes, p.b16 + (size_t)t * tile_elems, tile_bytes,
                   &b_full[bstage], pol_b);
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
      const int ksteps = p.kpad / 16;
      int bstage = 0;
      uint32_t bphase = 0;
      uint32_t acc_it = 0;
      int64_t it = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, it++) {
        const int64_t sc = item / nb;
        const int ab = (int)(it & 1);
        mbar_wait(&a_full[ab], (uint32_t)((it >> 1) & 1));
        tc_fence_after();
        const uint32_t a_addr = smem_u32(a_buf[ab]);
        const int64_t t0 = sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
        for (int64_t t = t0; t < t1; t++) {
          const uint32_t as = acc_it & 1u;
          mbar_wait(&acc_empty[as], ((acc_it >> 1) & 1u) ^ 1u);
          mbar_wait(&b_full[bstage], bphase);
          tc_fence_after();
          const uint32_t b_addr = smem_u32(b_buf + (size_t)bstage * L.b_bytes);
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const uint32_t d_tmem = tmem_base + as * 256 + h * 128;
            for (int kk = 0; kk < ksteps; kk++) {
              const uint64_t adesc =
                  umma_desc_kmajor_noswz(a_addr + h * tile_bytes + kk * 2 * lbo, lbo, sbo);
              const uint64_t bdesc = umma_desc_kmajor_noswz(b_addr + kk * 2 * lbo, lbo, sbo);
              tc_mma_bf16(d_tmem, adesc, bdesc, idesc, kk > 0 ? 1u : 0u);
            }
          }
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
        float v[128];
        const uint32_t taddr = tmem_base + (lane_base << 16) + as * 256 + h * 128;
        SJB_TMEM_LD32(taddr + 0, v, 0);
        SJB_TMEM_LD32(taddr + 32, v, 32);
        SJB_TMEM_LD32(taddr + 64, v, 64);
        SJB_TMEM_LD32(taddr + 96, v, 96);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[as]);
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
        const bool hit = row_ok && (m >= cutoff);
        if (__any_sync(0xffffffffu, hit)) {
          const int64_t j0 = t * kBN;
          const int64_t col_lim = p.n_b - j0;  // columns >= col_lim are padding
#pragma unroll
          for (int k = 0; k < 16; k++) {
            if (hit && g[k] >= cutoff) {
#pragma unroll
              for (int e = 0; e < 8; e++) {
                const int c = 8 * k + e;
                if (v[c] >= cutoff && c < col_lim) {
                  const unsigned act = __activemask();
                  const int leader = __ffs(act) - 1;
                  const unsigned rank = __popc(act & ((1u << lane) - 1u));
                  uint32_t base = 0;
                  if (lane == leader) {
                    const uint32_t np = (uint32_t)__popc(act);
                    base = atomicAdd(cta_cnt, np);
                    if (base + np < base) *cta_sat = 1u;
                  }
                  base = __shfl_sync(act, base, leader);
                  const uint64_t pos = (uint64_t)base + rank;
                  if (pos < seg_cap) seg[pos] = pack_pair(gi, (uint32_t)(j0 + c));
                }
              }
            }
          }
        }
      }
    }
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
