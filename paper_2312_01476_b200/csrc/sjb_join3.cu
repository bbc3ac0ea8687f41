// sjb_join3.cu -- fused threshold filter for wide embeddings (kpad > 128,
// e.g. BASELINE cfg4 d = 768), K-streaming.
//
// The resident-R design of sjb_join.cu needs the whole 256 x kpad R block in
// shared memory (384 KB at d = 768), so here both operands stream through the
// ring in K chunks of 64 elements: a stage = the R block's chunk (256 rows x
// 64, 32 KB) + the S tile's chunk (256 rows x 64, 32 KB), both contiguous in
// the [k-group][256][8] operand image.  Per chunk, 2 x 4 UMMA_128x256x16 (one
// per R half) accumulate into the two 256-column halves of TMEM; the output
// tile is 256 x 256 and K/64 chunks long (12 at d = 768: ~12k MMA cycles), so
// one accumulator stage suffices: each 256-column TMEM half is handed back
// (acc_empty[h]) as soon as the epilogue has drained it, so the next tile's
// first MMAs overlap the emission of the previous one.  Epilogue, candidate segments and the fused canonical recheck
// are those of sjb_join.cu.
#include "sjb_common.cuh"

namespace sjb {
namespace wide {

// At d >= 129 a 256 x 256 tile is >= 9 K-chunks of MMA work while the
// canonical recheck of its candidates is d-long chains from L2, so the warps
// lean to the recheck side.
constexpr int kEpiWarps = 8;
constexpr int kRecheckWarps = 10;
constexpr int kChunksPerWarp = 16 / kEpiWarps;  // 64-column chunks per half
constexpr int kThreads = 32 * (2 + kEpiWarps + kRecheckWarps);
constexpr int kKChunk = 64;                 // K elements per stage
constexpr int kChunkBytes = kTileRows * kKChunk * 2;  // 32 KB per operand

struct Params {
  const __nv_bfloat16* a16;
  const __nv_bfloat16* b16;
  int64_t n_a, n_b;
  int kpad;            // multiple of 64
  int n_ablk, n_btiles;  // 256-row blocks / tiles
  int tiles_per_chunk;
  int64_t n_items;
  int stages;
  float cutoff;
  uint64_t* cand;
  uint64_t seg_cap;
  unsigned long long* cta_count;
  const float* l32;
  const float* r32;
  int dim;
  float theta;
  uint32_t* sims_bits;
  uint32_t* rowcount;
  int debug;  // 1: recheck warps idle (filter timing only; results invalid)
};

__host__ __device__ inline uint32_t smem_bytes(int stages) {
  return (uint32_t)stages * 2 * kChunkBytes + (4 + 2 * stages) * 8 + 32;
}

__global__ void __launch_bounds__(kThreads, 1) filter_kernel(const Params p) {
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

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(acc_full, 1);
    mbar_init(&acc_empty[0], kEpiWarps);
    mbar_init(&acc_empty[1], kEpiWarps);
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    *cta_cnt = 0u;
    *cta_sat = 0u;
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
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int64_t rb = item % nb, sc = item / nb;
        const int64_t t0 = sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
        for (int64_t t = t0; t < t1; t++) {
          for (int c = 0; c < nchunks; c++) {
            mbar_wait(&empty[s], ph ^ 1u);
            mbar_arrive_expect_tx(&full[s], 2 * kChunkBytes);
            uint8_t* dst = ring + (size_t)s * 2 * kChunkBytes;
            bulk_g2s(dst, p.a16 + rb * tile_elems + c * chunk_elems, kChunkBytes, &full[s], pol_a);
            bulk_g2s(dst + kChunkBytes, p.b16 + t * tile_elems + c * chunk_elems, kChunkBytes,
                     &full[s], pol_b);
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
    const uint32_t idesc = umma_idesc_bf16_f32(128, 256);
    const uint32_t lbo = kTileRows * 16, sbo = 128;
    const uint64_t kstep = (2 * lbo) >> 4, half_step = (128 * 16) >> 4;
    const uint64_t ring_desc = umma_desc_kmajor_noswz(smem_u32(ring), lbo, sbo);
    const uint64_t stage_step = (2 * kChunkBytes) >> 4, b_off = kChunkBytes >> 4;
    int s = 0;
    uint32_t ph = 0, tile_it = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t sc = item / nb;
      const int64_t t0 = sc * p.tiles_per_chunk;
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
              tc_mma_bf16_elect(tmem_base + h * 256, ad + h * half_step + kk * kstep,
                                bd + kk * kstep, idesc, (c | kk) ? 1u : 0u);
          }
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
    // ------------------------------------------------------ recheck warps
    const uint64_t seg_cap = p.seg_cap;
    if (p.debug != 1)
      recheck_loop(p.cand + (uint64_t)blockIdx.x * seg_cap, p.sims_bits + (uint64_t)blockIdx.x * seg_cap,
                 seg_cap, cta_cnt, epi_done, (uint32_t)kEpiWarps, warp - 2 - kEpiWarps,
                 kRecheckWarps, p.l32, p.r32, p.dim, p.theta, p.rowcount);
  } else {
    // ---------------------------------------------------------- epilogue
    // warp (q, c): TMEM lanes 32q..32q+31 x column chunks c, c + 2 (64 each)
    // of BOTH halves; a half is handed back after its last chunk is loaded
    const int ew = warp - 2;
    const int cq0 = ew >> 2, q = warp & 3;
    const uint32_t lane_base = (uint32_t)q * 32;
    const float cutoff = p.cutoff;
    uint64_t* seg = p.cand + (uint64_t)blockIdx.x * p.seg_cap;
    const uint64_t seg_cap = p.seg_cap;
    uint32_t tile_it = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t rb = item % nb, sc = item / nb;
      const int64_t t0 = sc * p.tiles_per_chunk;
      const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
      for (int64_t t = t0; t < t1; t++, tile_it++) {
        mbar_wait(acc_full, tile_it & 1u);
        tc_fence_after();
#pragma unroll 1
        for (int h = 0; h < 2; h++) {
          const int64_t gi64 = rb * kTileRows + h * 128 + lane_base + lane;
#pragma unroll 1
          for (int k = 0; k < kChunksPerWarp; k++) {
            const int cq = cq0 + k * (kEpiWarps / 4);
            const uint32_t taddr = tmem_base + (lane_base << 16) + h * 256 + cq * 64;
            float v[64];
            SJB_TMEM_LD32(taddr, v, 0);
            SJB_TMEM_LD32(taddr + 32, v, 32);
            tc_wait_ld();
            if (k == kChunksPerWarp - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_relaxed(&acc_empty[h]);
            }
            const int64_t col_lim = p.n_b - t * kTileRows - cq * 64;
            emit_row_chunk64(v, gi64 < p.n_a, cutoff, (uint32_t)gi64,
                             (uint32_t)(t * kTileRows + cq * 64), col_lim, cta_cnt, cta_sat, seg,
                             seg_cap);
          }
        }
      }
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
  if (threadIdx.x == 0)
    p.cta_count[blockIdx.x] = *cta_sat ? ~0ull >> 1 : (unsigned long long)*cta_cnt;
}

}  // namespace wide
}  // namespace sjb
