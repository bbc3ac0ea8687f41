// sjb_join.cu -- the fused R.S^T threshold filter (the hot path).
//
// Replaces the reference's tile_similarity + threshold_scan pair
// (linalg.py:116-153 -> sj_tile_dot _kernelcore.c:273-296 + sj_scan_count/fill
// :300-323) with one persistent, warp-specialised tcgen05 kernel that never
// materialises the similarity matrix:
//
//   warp 0       S producer: 1-D bulk copies (TMA, cp.async.bulk) of pre-tiled
//                16-bit (bf16) operand tiles into a shared-memory ring (mbarriers)
//   warp 0 ln 1  R-block producer (resident operand, one copy per item)
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..17  epilogue: tcgen05.ld of the fp32 accumulators, 3-input max
//                pre-filter against (theta - band), candidate emission
//   warps 18..19 canonical recheck of the CTA's candidates (sequential fp32
//                fmaf dot == sj_dot_seq) while their rows are L2-resident
//
// Work item = (R block of 256 rows, S chunk of `tiles_per_chunk` 256-row
// tiles).  The R block stays resident in shared memory; the chunk's S tiles
// stream through a ring of B stages.  Each S tile is used by two M=128
// halves of the R block: 2 x (kpad/16) UMMA_128x256x16 instructions, one
// accumulator stage (128 lanes x 256 fp32 columns) per half; 2 stages = all
// 512 TMEM columns.  N = 256 keeps the operand reads at 96 B/cycle of the
// ~128 B/cycle shared-memory budget the SS-mode UMMA has (tools/mma_bench.cu:
// N <= 128 saturates it).  Items are ordered S-chunk-major so the CTAs
// resident at any moment share one S chunk in L2.
//
// Output: candidate pairs (i, j) with fp16 approx >= cutoff, packed as
// u64 (i << 32 | j) into per-CTA segments of `cand` (seg_cap each), counted in
// a shared-memory counter and published in cta_count[blockIdx.x].  A CTA
// whose segment overflows keeps counting, so the host can retry with the
// exact capacity (the schedule is static, so per-CTA counts are
// reproducible).  Every candidate is re-decided in canonical fp32 by the
// recheck warps: sims_bits[slot] = canonical sim (or kRejected), and
// rowcount[i] counts the matches of left row i for sjb_post.cu's bucketing.
#include "sjb_common.cuh"

#ifndef SJB_EMIT_RUNS
#define SJB_EMIT_RUNS 0
#endif

#ifndef SJB_PROFILE
#define SJB_PROFILE 0
#endif

namespace sjb {

constexpr int kEpiWarps = 16;
constexpr int kRecheckWarps = 2;
// 20 warps = 5 per SM sub-partition, which keeps the per-thread register cap
// at 96 (16K registers per SMSP); a 21st warp would force spills.
constexpr int kJoinThreads = 32 * (2 + kEpiWarps + kRecheckWarps);
constexpr int kBN = kTileRows;  // S rows per stage == UMMA N
constexpr int kUmmaN = 256;

struct JoinParams {
  const op16_t* a16;  // R operand image, n_ablk tiles
  const op16_t* b16;  // S operand image, n_btiles tiles
  int64_t n_a, n_b;          // valid rows
  int kpad;                  // padded K (multiple of 16, <= 128)
  int n_ablk;                // ceil(n_a / 256)
  int n_btiles;              // ceil(n_b / 256)
  int tiles_per_chunk;
  int tile_begin;            // first S tile of this launch (S-range launches)
  int append;                // 1: continue the segments of an earlier launch
  int defer;                 // 1: recheck warps idle; the row-grouped recheck runs later
  int64_t n_items;
  int stages;                // B stages
  int a_bufs;                // 1 or 2 resident-A buffers
  int a_tiles;               // 256-row operand tiles per resident R block (template ATILES)
  int ts;                    // 1: R block in tensor memory (sjb_join_ts.cu)
  float cutoff;
  const float* row_err;   // per-row band (or nullptr: uniform cutoff)
  const float* tile_err;
  float slack;
  uint64_t* cand;
  uint64_t seg_cap;
  unsigned long long* cta_count;
  // canonical recheck (fused): fp32 rows, decision and per-row match counts
  const float* l32;
  const float* r32;
  int dim;
  float theta;
  uint32_t* sims_bits;  // per candidate slot: canonical sim bits or kRejected
  uint32_t* rowcount;   // matches per left row
  int debug_mode;       // diagnostics: 0 normal, 1 no emission, 2 no TMEM drain
};

struct JoinSmemLayout {
  uint32_t tile_bytes;  // one 256-row operand tile
  uint32_t off_a, off_b, off_bar, total;
};

__host__ __device__ inline JoinSmemLayout join_smem_layout(int kpad, int stages, int a_bufs,
                                                          int a_tiles) {
  JoinSmemLayout L;
  L.tile_bytes = (uint32_t)kTileRows * kpad * 2;
  L.off_a = 0;
  L.off_b = a_bufs * a_tiles * L.tile_bytes;
  L.off_bar = L.off_b + stages * L.tile_bytes;
  // a_full[2] a_empty[2] acc_full[2] acc_empty[2] b_full[S] b_empty[S] + tmem slot
  // + candidate counter, wrap flag, finished-epilogue-warp count
  L.total = L.off_bar + (8 + 2 * stages) * 8 + 16 + 16;
  return L;
}

// KSTEPS = kpad / 16 UMMA k-steps (compile time so the issue loop is
// straight-line: each tcgen05.mma costs one descriptor add).  ATILES = 256-row
// operand tiles in the resident R block: each S tile is used by 2 * ATILES
// M=128 halves, so ATILES = 2 halves the S-tile TMA traffic (shared-memory
// writes and L2 reads) per MMA.
template <int KSTEPS, int ATILES>
__global__ void __launch_bounds__(kJoinThreads, 1) join_filter_kernel(const JoinParams p) {
  constexpr int kBM = kTileRows * ATILES;   // resident R rows per item
  constexpr int kHalves = 2 * ATILES;
  extern __shared__ __align__(1024) uint8_t smem[];
  const JoinSmemLayout L = join_smem_layout(p.kpad, p.stages, p.a_bufs, ATILES);
  uint8_t* a_buf = smem + L.off_a;
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
  uint32_t* epi_done = cta_cnt + 2;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; i++) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
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
  const int na = p.a_bufs;

  if (warp == 0 && lane == 1) {
    {
      // ------------------------------------------------- R-block producer
      // Separate thread from the S producer so the S ring keeps prefetching
      // across item boundaries while the next R block waits for its buffer.
      const uint64_t pol_a = policy_evict_last();
      int64_t it = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, it++) {
        const int64_t rb = item % nb;
        const int ab = (int)(it % na);
        mbar_wait(&a_empty[ab], (uint32_t)((it / na) & 1) ^ 1u);
        mbar_arrive_expect_tx(&a_full[ab], ATILES * tile_bytes);
        bulk_g2s(a_buf + (size_t)ab * ATILES * tile_bytes,
                 p.a16 + (size_t)rb * ATILES * tile_elems, ATILES * tile_bytes, &a_full[ab],
                 pol_a);
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      // -------------------------------------------------------- S producer
      const uint64_t pol_b = policy_evict_normal();
      int bstage = 0;
      uint32_t bphase = 0;
      int64_t it = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, it++) {
        const int64_t sc = item / nb;
        const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
        for (int64_t t = t0; t < t1; t++) {
          mbar_wait(&b_empty[bstage], bphase ^ 1u);
          if (p.debug_mode == 17 && it > 0) {
            mbar_arrive(&b_full[bstage]);  // diagnostics: no B traffic after the first item
          } else {
            mbar_arrive_expect_tx(&b_full[bstage], tile_bytes);
            bulk_g2s(b_buf + (size_t)bstage * tile_bytes, p.b16 + (size_t)t * tile_elems,
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
    {
      // ------------------------------------------------------- MMA issuer
      // whole warp, warp-uniform control flow; one elected lane issues each
      // tcgen05 op (a single divergent lane costs an ELECT/R2UR sequence
      // per MMA and made the issue the critical path)
      const uint32_t idesc = umma_idesc_f16_f32(128, kUmmaN, true);
      const uint32_t lbo = kTileRows * 16;  // 256-row operand: distance between k-groups
      const uint32_t sbo = 128;             // distance between 8-row core-matrix groups
      // a k-step advances the start address by 2 k-groups = 2 * lbo bytes;
      // the second M half starts 128 rows (= 16 core-matrix groups) later
      const uint64_t kstep = (2 * lbo) >> 4;
      const uint64_t half_step = (128 * 16) >> 4;
      const uint64_t a_desc_base = umma_desc_kmajor_noswz(smem_u32(a_buf), lbo, sbo);
      const uint64_t b_desc_base = umma_desc_kmajor_noswz(smem_u32(b_buf), lbo, sbo);
      const uint64_t tile_step = tile_bytes >> 4;
      int bstage = 0;
      uint32_t bphase = 0;
      uint32_t acc_it = 0;
      int64_t it = 0;
      // diagnostics (build with -DSJB_PROFILE=1, run with SJB_DEBUG_MODE=9):
      // wait-time attribution of the MMA thread
      const bool dbg = SJB_PROFILE && p.debug_mode == 9;
      long long w_a = 0, w_b = 0, w_e = 0;
      const long long c_start = clock64();
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, it++) {
        const int64_t sc = item / nb;
        const int ab = (int)(it % na);
        long long c0 = dbg ? clock64() : 0;
        mbar_wait(&a_full[ab], (uint32_t)((it / na) & 1));
        if (dbg) w_a += clock64() - c0;
        tc_fence_after();
        const uint64_t ad = a_desc_base + (uint64_t)ab * ATILES * tile_step;
        const int64_t t0 = p.tile_begin + sc * p.tiles_per_chunk;
        const int64_t t1 = mn<int64_t>(t0 + p.tiles_per_chunk, p.n_btiles);
        for (int64_t t = t0; t < t1; t++) {
          if (dbg) c0 = clock64();
          mbar_wait(&b_full[bstage], bphase);
          if (dbg) w_b += clock64() - c0;
          const uint64_t bd = b_desc_base + (uint64_t)bstage * tile_step;
#pragma unroll
          for (int h = 0; h < kHalves; h++) {
            const uint32_t as = acc_it & 1u;
            if (dbg) c0 = clock64();
            mbar_wait(&acc_empty[as], ((acc_it >> 1) & 1u) ^ 1u);
            if (dbg) w_e += clock64() - c0;
            tc_fence_after();
            const uint32_t d = tmem_base + as * kUmmaN;
            const uint64_t adh = ad + (h >> 1) * tile_step + (h & 1) * half_step;
#pragma unroll
            for (int kk = 0; kk < KSTEPS; kk++)
              tc_mma_f16_elect(d, adh + kk * kstep, bd + kk * kstep, idesc, kk > 0 ? 1u : 0u);
            tc_commit_elect(&acc_full[as]);
            acc_it++;
          }
          tc_commit_elect(&b_empty[bstage]);
          if (++bstage == p.stages) {
            bstage = 0;
            bphase ^= 1u;
          }
        }
        tc_commit_elect(&a_empty[ab]);
      }
      if (dbg && blockIdx.x < 3 && lane == 0)
        printf("[dbg] cta %d mma: total %lld  wait_a %lld  wait_b %lld  wait_acc_empty %lld\n",
               blockIdx.x, clock64() - c_start, w_a, w_b, w_e);
    }
  } else if (warp >= 2 + kEpiWarps) {
    // ------------------------------------------------------ recheck warps
    // Re-decide every candidate of this CTA in canonical fp32 while the S
    // chunk it came from is still L2-resident.  Warp w owns 32-slot blocks
    // w, w + kRecheckWarps, ...; a block is processed once reserved (or once
    // the epilogue has finished); each lane waits for its slot to be written
    // (slots start as kEmptySlot).
    const int rw = warp - 2 - kEpiWarps;
    const uint64_t seg_cap = p.seg_cap;
    const uint64_t* seg = p.cand + (uint64_t)blockIdx.x * seg_cap;
    uint32_t* sims = p.sims_bits + (uint64_t)blockIdx.x * seg_cap;
    volatile uint32_t* vcnt = cta_cnt;
    volatile uint32_t* vdone = epi_done;
    if (p.debug_mode != 5 && !p.defer)  // (diagnostics: 5 = emit, no recheck, results invalid)
      recheck_loop(seg, sims, seg_cap, vcnt, vdone, (uint32_t)kEpiWarps, rw, kRecheckWarps,
                   p.l32, p.r32, p.dim, p.theta, p.rowcount,
                   p.append ? (uint64_t)p.cta_count[blockIdx.x] : 0ull);
  } else {
    // ---------------------------------------------------------- epilogue
    // 16 warps in two stage groups: group g drains accumulator stage g (the
    // R block's half g) of every S tile, so each warp has two MMA stage times
    // per stage it drains.  Warp (q, c) of a group reads TMEM lanes
    // 32q..32q+31 (R rows) x columns 128c..128c+127 (S rows) as two x64
    // loads; the stage is released after the second load, and a hit lane's
    // candidate masks are built while its values are live but emitted after
    // the release, so hits never hold the accumulator.  The slack before the
    // MMA waits is a whole stage plus the other group's stage, which absorbs
    // the emission of hit chunks (tools/power_modes.py).
    const int ew = warp - 2;
    const int grp = ew >> 3;          // accumulator stage drained (halves grp, grp + 2, ..)
    const int cq = (ew >> 2) & 1;     // 128-column half of the 256-column stage
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const uint32_t lane_base = (uint32_t)q * 32;
    uint64_t* seg = p.cand + (uint64_t)blockIdx.x * p.seg_cap;
    const uint64_t seg_cap = p.seg_cap;
    const bool edbg = SJB_PROFILE && p.debug_mode == 9 && blockIdx.x < 3 && (ew == 0 || ew == 15);
    long long e_wait = 0, e_drain = 0, e_mark = 0;
    const long long e_start = clock64();
    const uint32_t tbase = tmem_base + (lane_base << 16) + (uint32_t)grp * kUmmaN + (uint32_t)cq * 128;
    const bool no_drain = p.debug_mode == 2 || p.debug_mode >= 16;   // diagnostics
    const bool no_emit = p.debug_mode == 1;
    const bool per_row = p.row_err != nullptr;
    // columns of a 64-column chunk that are >= cutoff, inside groups of 8
    // whose maximum hit (hit lanes only)
    auto chunk_mask = [&](const float* v, const float* g, float cutoff, uint32_t& mk0,
                          uint32_t& mk1) {
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
    };
    // one warp's candidates: slots reserved with one shared atomic; then
    // round r writes the r-th candidate of every lane that still has one to
    // consecutive slots (rank among the round's lanes), so a round is one
    // coalesced store (SJB_EMIT_RUNS=1 at build: per-lane runs, round 1).
    // Nothing downstream depends on the order inside a warp's slot range.
    auto emit = [&](const uint32_t (&mk)[4], uint32_t gi, uint32_t j0) {
      const uint32_t cnt = __popc(mk[0]) + __popc(mk[1]) + __popc(mk[2]) + __popc(mk[3]);
#if SJB_EMIT_RUNS
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
#pragma unroll
      for (int wd = 0; wd < 4; wd++) {
        uint32_t w = mk[wd];
        while (w) {
          const int b = __ffs(w) - 1;
          w &= w - 1;
          if (pos < seg_cap) seg[pos] = pack_pair(gi, j0 + 32 * wd + b);
          pos++;
        }
      }
#else
      const uint32_t wtot = __reduce_add_sync(0xffffffffu, cnt);
      uint32_t base = 0;
      if (lane == 0) {
        base = atomicAdd(cta_cnt, wtot);
        if (base + wtot < base) *cta_sat = 1u;
      }
      uint64_t run = __shfl_sync(0xffffffffu, base, 0);
      const uint32_t lt = lanemask_lt();
      uint32_t w0 = mk[0], w1 = mk[1], w2 = mk[2], w3 = mk[3];
      for (;;) {
        const bool act = (w0 | w1 | w2 | w3) != 0u;
        const uint32_t am = __ballot_sync(0xffffffffu, act);
        if (am == 0u) break;
        if (act) {
          int col;
          if (w0) { col = __ffs(w0) - 1; w0 &= w0 - 1; }
          else if (w1) { col = 32 + __ffs(w1) - 1; w1 &= w1 - 1; }
          else if (w2) { col = 64 + __ffs(w2) - 1; w2 &= w2 - 1; }
          else { col = 96 + __ffs(w3) - 1; w3 &= w3 - 1; }
          const uint64_t pos = run + __popc(am & lt);
          if (pos < seg_cap) seg[pos] = pack_pair(gi, j0 + col);
        }
        run += __popc(am);
      }
#endif
    };
    uint32_t tph = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t rb = item % nb, sc = item / nb;
      const int t0 = p.tile_begin + (int)sc * p.tiles_per_chunk;
      const int t1 = mn<int>(t0 + p.tiles_per_chunk, p.n_btiles);
      // per-row band: cutoff = max(cutoff, theta - slack - (1+1e-6)(ex + ey)
      // - ex*ey) = max(cutoff, cA - cB*ey); the 2e-6 in `slack` covers the
      // fp32 evaluation of either form.  This group's halves of the R block
      // are h = grp (and grp + 2 when ATILES = 2), kept as scalars and
      // selected per use so the stage body is emitted once (a copy per half
      // doubled the epilogue's code: 17.1 vs 16.5 ms)
      const int64_t g0 = rb * kBM + grp * 128 + lane_base + lane, g1 = g0 + 256;
      const bool rok0 = g0 < p.n_a && !no_emit, rok1 = g1 < p.n_a && !no_emit;
      const float ex0 = load_err(p.row_err, g0, p.n_a);
      const float ex1 = ATILES > 1 ? load_err(p.row_err, g1, p.n_a) : 0.0f;
      const float cA0 = per_row ? p.theta - p.slack - 1.000001f * ex0 : p.cutoff;
      const float cA1 = per_row ? p.theta - p.slack - 1.000001f * ex1 : p.cutoff;
      const float cB0 = per_row ? 1.000001f + ex0 : 0.0f, cB1 = per_row ? 1.000001f + ex1 : 0.0f;
      for (int t = t0; t < t1; t++) {
        // issued before the accumulator wait: its latency hides behind it
        const float ey = per_row ? __ldg(p.tile_err + t) : 0.0f;
#pragma unroll 1
        for (int hh = 0; hh < ATILES; hh++) {
          const bool h1 = hh != 0;
          const long long e0 = edbg ? clock64() : 0;
          mbar_wait(&acc_full[grp], tph);
          tph ^= 1u;
          if (edbg) { const long long e1 = clock64(); e_wait += e1 - e0; e_mark = e1; }
          tc_fence_after();
          if (no_drain) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[grp]);
            continue;
          }
          const float cutoff = fmaxf(p.cutoff, fmaf(h1 ? -cB1 : -cB0, ey, h1 ? cA1 : cA0));
          uint32_t mk[4] = {0u, 0u, 0u, 0u};
          bool any_hit = false;
#pragma unroll
          for (int c = 0; c < 2; c++) {
            float v[64];
            SJB_TMEM_LD64(tbase + c * 64, v);
            tc_wait_ld();
            if (c == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_relaxed(&acc_empty[grp]);
              if (edbg) e_drain += clock64() - e_mark;
            }
            // group maxima over 8 columns, then the 64-column maximum
            float g[8];
#pragma unroll
            for (int k = 0; k < 8; k++) {
              const float* x = v + 8 * k;
              g[k] = fmax3(fmax3(x[0], x[1], x[2]), fmax3(x[3], x[4], x[5]), fmaxf(x[6], x[7]));
            }
            const float m =
                fmax3(fmax3(g[0], g[1], g[2]), fmax3(g[3], g[4], g[5]), fmaxf(g[6], g[7]));
            const bool hit = (h1 ? rok1 : rok0) && (m >= cutoff);
            if (__any_sync(0xffffffffu, hit)) {
              if (hit) chunk_mask(v, g, cutoff, mk[2 * c], mk[2 * c + 1]);
              any_hit = true;
            }
          }
          if (any_hit) {
            const int64_t col_lim = p.n_b - (int64_t)t * kBN - cq * 128;  // >= col_lim: padding
            if (col_lim < 128) {
#pragma unroll
              for (int wd = 0; wd < 4; wd++) {
                const int64_t cl = col_lim - 32 * wd;
                mk[wd] &= cl >= 32 ? ~0u : (cl <= 0 ? 0u : ((1u << cl) - 1u));
              }
            }
            emit(mk, (uint32_t)(h1 ? g1 : g0), (uint32_t)(t * kBN + cq * 128));
          }
        }
      }
    }
    if (edbg && lane == 0)
      printf("[dbg] cta %d epi warp %d: total %lld  wait_acc_full %lld  drain %lld\n",
             blockIdx.x, ew, clock64() - e_start, e_wait, e_drain);
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

}  // namespace sjb
