// sjb_common.cuh -- shared constants and sm_100a PTX wrappers (mbarrier, bulk
// copy, tcgen05) for the simjoin-b200 kernels.  Hand-written inline PTX; no
// CUTLASS/CuTe.  Compile only with -gencode arch=compute_100a,code=sm_100a.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace sjb {

// 16-bit tensor-core operands, raw storage; the format follows the path
// (DESIGN.md section 2):
//  * kpad <= 128 (the resident-R filter): bf16.  Same UMMA rate as fp16, but
//    the tensor pipe draws less power per MMA, and the filter runs at the
//    board power cap: cfg2 15.8 vs 16.5 ms sustained (MMA-only 13.6 vs
//    14.65) for 8% more candidates, which the fused recheck absorbs.
//  * kpad > 128 (the K-streaming wide filter): fp16.  Its 11-bit significand
//    rounds 8x finer, so the band admits far fewer non-matches (cfg4: 5.3e8
//    vs 7.5e8 candidates), and there the canonical recheck dominates.
using op16_t = uint16_t;
__host__ __device__ constexpr bool op_is_bf16(int kpad) { return kpad <= 128; }
__device__ __forceinline__ op16_t to_op16(float x, bool bf) {
  return bf ? __bfloat16_as_ushort(__float2bfloat16_rn(x)) : __half_as_ushort(__float2half_rn(x));
}
__device__ __forceinline__ float from_op16(op16_t h, bool bf) {
  return bf ? __bfloat162float(__ushort_as_bfloat16(h)) : __half2float(__ushort_as_half(h));
}


// Rows per 16-bit operand tile.  Both relations are stored as a sequence of
// 256-row tiles in the UMMA canonical K-major no-swizzle layout
// ([k-group of 8 elements][row][8 elements], 16 B core-matrix rows), so one
// 1-D bulk copy moves a whole tile into shared memory and the tensor core
// reads it directly (as one N=256 operand, or as two M=128 halves at a
// 2 KB offset).  See DESIGN.md "HBM layout".
constexpr int kTileRows = 256;

__host__ __device__ inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
__host__ __device__ inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

// Element offset of (row, k) inside the tiled 16-bit image of a relation with
// `kpad` padded columns.
__host__ __device__ inline int64_t tiled_offset(int64_t row, int64_t k, int64_t kpad) {
  int64_t t = row / kTileRows, r = row % kTileRows;
  return t * (kTileRows * kpad) + (k / 8) * (kTileRows * 8) + r * 8 + (k % 8);
}

// Pack (i, j) offsets into the 64-bit candidate word (left in the high half).
__host__ __device__ inline uint64_t pack_pair(uint32_t i, uint32_t j) {
  return (uint64_t(i) << 32) | uint64_t(j);
}

template <class T>
__host__ __device__ __forceinline__ T mn(T a, T b) { return a < b ? a : b; }
template <class T>
__host__ __device__ __forceinline__ T mx(T a, T b) { return a < b ? b : a; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Relaxed arrive: no release ordering of this thread's prior memory ops
// (used where only tcgen05 ordering matters, so outstanding global stores
// of the epilogue never delay the hand-off).
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SJB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SJB_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------- bulk copy (TMA, 1-D)
// Global -> shared bulk copy completing `bytes` of transaction count on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ldg4_hint(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
// 32-byte read-only load (LDG.256, sm_100): one full sector per lane
struct f8 {
  float v[8];
};
__device__ __forceinline__ f8 ldg8_hint(const float* p, uint64_t pol) {
  f8 r;
  asm volatile("ld.global.nc.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                 "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------------------ tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Arrive on `bar` once all previously issued tcgen05 ops of this thread finish.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (fp16 in, fp32 accumulate).
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-uniform variants: the whole warp executes the call, one elected lane
// issues (keeps descriptors in uniform registers; no per-MMA ELECT loop).
__device__ __forceinline__ void tc_mma_f16_elect(uint32_t d_tmem, uint64_t a_desc,
                                                  uint64_t b_desc, uint32_t idesc,
                                                  uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 lanes x 32 consecutive fp32 columns: thread t of the warp gets lane
// (taddr.lane + t), columns [taddr.col, taddr.col + 32).
// 32 lanes x 64 consecutive fp32 columns in one instruction.
#define SJB_TMEM_LD64(taddr, v)                                                             \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"     \
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]), "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31]), "=f"(v[32]), "=f"(v[33]), "=f"(v[34]), "=f"(v[35]), "=f"(v[36]), "=f"(v[37]), "=f"(v[38]), "=f"(v[39]), "=f"(v[40]), "=f"(v[41]), "=f"(v[42]), "=f"(v[43]), "=f"(v[44]), "=f"(v[45]), "=f"(v[46]), "=f"(v[47]), "=f"(v[48]), "=f"(v[49]), "=f"(v[50]), "=f"(v[51]), "=f"(v[52]), "=f"(v[53]), "=f"(v[54]), "=f"(v[55]), "=f"(v[56]), "=f"(v[57]), "=f"(v[58]), "=f"(v[59]), "=f"(v[60]), "=f"(v[61]), "=f"(v[62]), "=f"(v[63])           \
               : "r"(taddr))

#define SJB_TMEM_LD32(taddr, v, o)                                                          \
  asm volatile(                                                                             \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                             \
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                             \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"           \
      : "=f"(v[o + 0]), "=f"(v[o + 1]), "=f"(v[o + 2]), "=f"(v[o + 3]), "=f"(v[o + 4]),     \
        "=f"(v[o + 5]), "=f"(v[o + 6]), "=f"(v[o + 7]), "=f"(v[o + 8]), "=f"(v[o + 9]),     \
        "=f"(v[o + 10]), "=f"(v[o + 11]), "=f"(v[o + 12]), "=f"(v[o + 13]),                 \
        "=f"(v[o + 14]), "=f"(v[o + 15]), "=f"(v[o + 16]), "=f"(v[o + 17]),                 \
        "=f"(v[o + 18]), "=f"(v[o + 19]), "=f"(v[o + 20]), "=f"(v[o + 21]),                 \
        "=f"(v[o + 22]), "=f"(v[o + 23]), "=f"(v[o + 24]), "=f"(v[o + 25]),                 \
        "=f"(v[o + 26]), "=f"(v[o + 27]), "=f"(v[o + 28]), "=f"(v[o + 29]),                 \
        "=f"(v[o + 30]), "=f"(v[o + 31])                                                    \
      : "r"(taddr))

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE canonical layout:
// core matrix = 8 rows x 16 B contiguous; `lbo` = byte distance between
// core matrices adjacent along K, `sbo` = byte distance between 8-row groups.
__device__ __forceinline__ uint64_t umma_desc_kmajor_noswz(uint32_t smem_addr, uint32_t lbo,
                                                          uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((smem_addr & 0x3FFFF) >> 4);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // descriptor version (sm_100)
  // base_offset = 0, lbo_mode = 0, layout_type (bits 61-63) = 0 (SWIZZLE_NONE)
  return d;
}

// Instruction descriptor: kind::f16, A=B=f16 (or bf16), D=f32, both
// K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_f16_f32(int M, int N, bool bf16 = false) {
  return (1u << 4)                      // D format f32
         | ((bf16 ? 1u : 0u) << 7)      // A format: 0 f16, 1 bf16
         | ((bf16 ? 1u : 0u) << 10)     // B format
         | (uint32_t(N >> 3) << 17)     // N / 8
         | (uint32_t(M >> 4) << 24);    // M / 16
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// Canonical similarity: sequential fp32 fused multiply-add over d, exactly
// the reference's sj_dot_seq with MADD = fmaf (_kernelcore.c:21-25, 101-106).
__device__ __forceinline__ float dot_seq_dev(const float* __restrict__ a,
                                             const float* __restrict__ b, int dim) {
  float acc = 0.0f;
  if ((dim & 3) == 0 &&
      ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0) {
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    for (int d = 0; d < (dim >> 2); d++) {
      const float4 x = __ldg(a4 + d), y = __ldg(b4 + d);
      acc = __fmaf_rn(x.x, y.x, acc);
      acc = __fmaf_rn(x.y, y.y, acc);
      acc = __fmaf_rn(x.z, y.z, acc);
      acc = __fmaf_rn(x.w, y.w, acc);
    }
  } else {
    for (int d = 0; d < dim; d++) acc = __fmaf_rn(__ldg(a + d), __ldg(b + d), acc);
  }
  return acc;
}

// Two canonical similarities with their (independent) sequential chains
// interleaved, so the FMA latency of one hides behind the other.  Each chain
// is exactly dot_seq_dev.
__device__ __forceinline__ void dot_seq2_dev(const float* __restrict__ a0,
                                             const float* __restrict__ b0,
                                             const float* __restrict__ a1,
                                             const float* __restrict__ b1, int dim, float& r0,
                                             float& r1) {
  float c0 = 0.0f, c1 = 0.0f;
  if ((dim & 3) == 0 && ((reinterpret_cast<uintptr_t>(a0) | reinterpret_cast<uintptr_t>(b0) |
                          reinterpret_cast<uintptr_t>(a1) | reinterpret_cast<uintptr_t>(b1)) &
                         15) == 0) {
    const float4 *x4 = reinterpret_cast<const float4*>(a0), *y4 = reinterpret_cast<const float4*>(b0);
    const float4 *u4 = reinterpret_cast<const float4*>(a1), *w4 = reinterpret_cast<const float4*>(b1);
#pragma unroll 5
    for (int d = 0; d < (dim >> 2); d++) {
      const float4 x = __ldg(x4 + d), y = __ldg(y4 + d), u = __ldg(u4 + d), w = __ldg(w4 + d);
      c0 = __fmaf_rn(x.x, y.x, c0);
      c1 = __fmaf_rn(u.x, w.x, c1);
      c0 = __fmaf_rn(x.y, y.y, c0);
      c1 = __fmaf_rn(u.y, w.y, c1);
      c0 = __fmaf_rn(x.z, y.z, c0);
      c1 = __fmaf_rn(u.z, w.z, c1);
      c0 = __fmaf_rn(x.w, y.w, c0);
      c1 = __fmaf_rn(u.w, w.w, c1);
    }
  } else {
    for (int d = 0; d < dim; d++) {
      c0 = __fmaf_rn(__ldg(a0 + d), __ldg(b0 + d), c0);
      c1 = __fmaf_rn(__ldg(a1 + d), __ldg(b1 + d), c1);
    }
  }
  r0 = c0;
  r1 = c1;
}

// Load that bypasses L1 (sees another warp's completed global stores).
__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Marks a candidate slot whose canonical similarity fell below theta.
constexpr uint32_t kRejected = 0x7fc00001u;  // a NaN payload no similarity can have
constexpr uint64_t kEmptySlot = ~0ull;         // candidate slot not yet written

// Epilogue reduce + emission for one warp's 32 rows x 64 accumulator columns
// (warp-synchronous; every lane calls it): group maxima over 8 columns with
// 3-input max, a warp vote, and -- only if some lane has a column >= cutoff --
// per-lane 64-bit hit masks, one warp scan + one shared atomic reserving the
// warp's candidate slots, and per-lane stores of (row, j0 + column) pairs.
// Columns >= col_lim are padding and never emitted.
// Filter cutoff of R row i against the 256-row S tile t256.  Without error
// arrays: the uniform theta - band.  With them:
// |approx - canonical| <= slack + (1+1e-6)(e_i + E_t) + e_i E_t, where e_i
// bounds ||fp16(x_i) - x_i|| and E_t the same over the S tile (Cauchy-Schwarz
// on the rounding errors; slack covers both fp32 accumulations and this fp32
// evaluation), so the cutoff can be raised to theta minus that bound.
__device__ __forceinline__ float row_cutoff(float cutoff, float theta, float slack,
                                            const float* row_err, const float* tile_err,
                                            int64_t i, int64_t n_a, int64_t t256) {
  if (row_err == nullptr) return cutoff;
  const float ex = i < n_a ? __ldg(row_err + i) : 0.0f;
  const float ey = __ldg(tile_err + t256);
  const float b = slack + 1.000001f * (ex + ey) + ex * ey;
  return fmaxf(cutoff, theta - b);
}

// The same cutoff from already-loaded errors (ex of the row, ey of the tile):
// kernels load them ahead of the accumulator wait so the latency is hidden.
__device__ __forceinline__ float cutoff_from(float cutoff, float theta, float slack, float ex,
                                             float ey) {
  const float b = slack + 1.000001f * (ex + ey) + ex * ey;
  return fmaxf(cutoff, theta - b);
}
__device__ __forceinline__ float load_err(const float* e, int64_t i, int64_t n) {
  return (e != nullptr && i < n) ? __ldg(e + i) : 0.0f;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <int CW>   // chunk width: 64 columns, or 32
__device__ __forceinline__ void emit_row_chunk(const float* v, bool row_ok, float cutoff,
                                               uint32_t gi, uint32_t j0, int64_t col_lim,
                                               uint32_t* cta_cnt, uint32_t* cta_sat,
                                               uint64_t* seg, uint64_t seg_cap) {
  static_assert(CW == 64 || CW == 32, "chunk width");
  constexpr int kG = CW / 8;
  const int lane = threadIdx.x & 31;
  float g[kG];
#pragma unroll
  for (int k = 0; k < kG; k++) {
    const float* x = v + 8 * k;
    g[k] = fmax3(fmax3(x[0], x[1], x[2]), fmax3(x[3], x[4], x[5]), fmaxf(x[6], x[7]));
  }
  float m;
  if (CW == 64)
    m = fmax3(fmax3(g[0], g[1], g[2]), fmax3(g[3], g[4], g[5]), fmaxf(g[kG - 2], g[kG - 1]));
  else
    m = fmaxf(fmax3(g[0], g[1], g[2]), g[3]);
  const bool hit = row_ok && m >= cutoff;
  if (!__any_sync(0xffffffffu, hit)) return;
  uint32_t mk0 = 0, mk1 = 0;
  if (hit) {
#pragma unroll
    for (int k = 0; k < kG; k++) {
      if (g[k] >= cutoff) {
        uint32_t b = 0;
#pragma unroll
        for (int e = 0; e < 8; e++) b |= (v[8 * k + e] >= cutoff ? 1u : 0u) << e;
        if (k < 4) mk0 |= b << (8 * k);
        else mk1 |= b << (8 * (k - 4));
      }
    }
    if (col_lim < CW) {
      const int cl = col_lim < 0 ? 0 : (int)col_lim;
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
  uint32_t w = mk0;
  while (w) {
    const int b = __ffs(w) - 1;
    w &= w - 1;
    if (pos < seg_cap) seg[pos] = pack_pair(gi, j0 + b);
    pos++;
  }
  if (CW == 64) {
    w = mk1;
    while (w) {
      const int b = __ffs(w) - 1;
      w &= w - 1;
      if (pos < seg_cap) seg[pos] = pack_pair(gi, j0 + 32 + b);
      pos++;
    }
  }
}
__device__ __forceinline__ void emit_row_chunk64(const float* v, bool row_ok, float cutoff,
                                                 uint32_t gi, uint32_t j0, int64_t col_lim,
                                                 uint32_t* cta_cnt, uint32_t* cta_sat,
                                                 uint64_t* seg, uint64_t seg_cap) {
  emit_row_chunk<64>(v, row_ok, cutoff, gi, j0, col_lim, cta_cnt, cta_sat, seg, seg_cap);
}

// Tolerance emission (raw-operand wide filter, sims_mode 1): the same hit
// masks and slot reservation as emit_row_chunk64 (every pair with approx >=
// cutoff gets a slot), but each slot's sim is written here: approx itself for
// pairs at or above hi_cut (final matches -- |approx - canonical| < band, so
// the canonical decision is certain -- counted into the row), kPending for
// the band pairs, whose slots are appended to the CTA's pending list.
constexpr uint32_t kPending = 0x7fc00002u;   // a NaN payload: recheck pending

// Returns the chunk's final matches of this lane's row (the caller adds them
// to the row count once per work item: one global atomic per row and item
// instead of one per chunk -- every epilogue warp of a CTA works on the same
// 256 rows, so per-chunk atomics on them serialise).  `scr` is this lane's
// 32-float shared scratch row: per 32-column half with hits, the 8-column
// groups holding hits are parked there, so the hit loop reads the similarity
// of a dynamic column without spilling v[] (static indices only) and the
// code stays as compact as emit_row_chunk64's.
template <int CW>   // chunk width: 64 columns, or 32 (16 epilogue warps: half the live registers)
__device__ __forceinline__ uint32_t emit_row_chunk_tol(
    const float* v, bool row_ok, float cutoff, float hi_cut, uint32_t gi, uint32_t j0,
    int64_t col_lim, uint32_t* cta_cnt, uint32_t* cta_sat, uint64_t* seg, uint64_t seg_cap,
    uint32_t* sims, uint32_t* pend_cnt, uint32_t* pend, float* scr) {
  static_assert(CW == 64 || CW == 32, "chunk width");
  constexpr int kG = CW / 8;
  const int lane = threadIdx.x & 31;
  float g[kG];
#pragma unroll
  for (int k = 0; k < kG; k++) {
    const float* x = v + 8 * k;
    g[k] = fmax3(fmax3(x[0], x[1], x[2]), fmax3(x[3], x[4], x[5]), fmaxf(x[6], x[7]));
  }
  float m;
  if (CW == 64)
    m = fmax3(fmax3(g[0], g[1], g[2]), fmax3(g[3], g[4], g[5]), fmaxf(g[kG - 2], g[kG - 1]));
  else
    m = fmaxf(fmax3(g[0], g[1], g[2]), g[3]);
  const bool hit = row_ok && m >= cutoff;
  if (!__any_sync(0xffffffffu, hit)) return 0u;
  uint32_t mk0 = 0, mk1 = 0;
  if (hit) {
#pragma unroll
    for (int k = 0; k < kG; k++) {
      if (g[k] >= cutoff) {
        uint32_t b = 0;
#pragma unroll
        for (int e = 0; e < 8; e++) b |= (v[8 * k + e] >= cutoff ? 1u : 0u) << e;
        if (k < 4) mk0 |= b << (8 * k);
        else mk1 |= b << (8 * (k - 4));
      }
    }
    if (col_lim < CW) {
      const int cl = col_lim < 0 ? 0 : (int)col_lim;
      mk0 &= cl >= 32 ? ~0u : ((1u << cl) - 1u);
      mk1 &= cl <= 32 ? 0u : ((1u << (cl - 32)) - 1u);
    }
  }
  const uint32_t wtot = __reduce_add_sync(0xffffffffu, __popc(mk0) + __popc(mk1));
  uint32_t base = 0;
  if (lane == 0) {
    base = atomicAdd(cta_cnt, wtot);
    if (base + wtot < base) *cta_sat = 1u;
  }
  uint64_t run = __shfl_sync(0xffffffffu, base, 0);
  const uint32_t lt = lanemask_lt();
  uint32_t finals = 0;
#pragma unroll
  for (int hh = 0; hh < CW / 32; hh++) {
    uint32_t w = hh ? mk1 : mk0;
    if (w != 0u) {
#pragma unroll
      for (int k = 0; k < 4; k++)
        if ((w >> (8 * k)) & 0xFFu) {
#pragma unroll
          for (int e = 0; e < 8; e++) scr[8 * k + e] = v[32 * hh + 8 * k + e];
        }
    }
    // rounds of lane-interleaved, consecutive slots: round i writes the i-th
    // hit of every lane that still has one, so each round is one coalesced
    // store instead of 32 scattered ones (the pending recheck and the row
    // bucketing are order-free; the canonical-sims group recheck prefers a
    // row's candidates adjacent, so emit_row_chunk64 keeps per-lane runs)
    for (;;) {
      const bool act = w != 0u;
      const uint32_t am = __ballot_sync(0xffffffffu, act);
      if (am == 0u) break;
      if (act) {
        const int b = __ffs(w) - 1;
        w &= w - 1;
        const uint64_t pos = run + __popc(am & lt);
        if (pos < seg_cap) {
          const float x = scr[b];
          seg[pos] = pack_pair(gi, j0 + 32 * hh + b);
          const bool fin = x >= hi_cut;
          sims[pos] = fin ? __float_as_uint(x) : kPending;
          finals += fin ? 1u : 0u;
          if (!fin) pend[atomicAdd(pend_cnt, 1u)] = (uint32_t)pos;
        }
      }
      run += __popc(am);
    }
  }
  return finals;
}
__device__ __forceinline__ uint32_t emit_row_chunk64_tol(
    const float* v, bool row_ok, float cutoff, float hi_cut, uint32_t gi, uint32_t j0,
    int64_t col_lim, uint32_t* cta_cnt, uint32_t* cta_sat, uint64_t* seg, uint64_t seg_cap,
    uint32_t* sims, uint32_t* pend_cnt, uint32_t* pend, float* scr) {
  return emit_row_chunk_tol<64>(v, row_ok, cutoff, hi_cut, gi, j0, col_lim, cta_cnt, cta_sat, seg,
                                seg_cap, sims, pend_cnt, pend, scr);
}

// One canonical recheck of a written candidate slot.
__device__ __forceinline__ uint64_t wait_slot(const uint64_t* slot) {
  uint64_t u;
  do {
    u = ld_volatile_u64(slot);
  } while (u == kEmptySlot);
  return u;
}

// Recheck warp loop shared by the filter kernels: warp `rw` of `nrw` owns
// 64-slot blocks rw, rw + nrw, ... of this CTA's candidate segment; a block is
// processed once fully reserved (or once all `n_epi` epilogue warps are done);
// each lane re-decides two slots with interleaved canonical chains, writes
// the canonical sim bits (or kRejected) and counts kept matches per left row.
// Segment count a filter launch starts from: 0, or (append) where the
// previous launch over other S tiles of the same join stopped.
__device__ __forceinline__ void init_segment_count(const unsigned long long* cta_count, bool append,
                                                   uint32_t* cnt, uint32_t* sat) {
  const unsigned long long c0 = append ? cta_count[blockIdx.x] : 0ull;
  *cnt = c0 > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)c0;
  *sat = c0 > 0xFFFFFFFFull ? 1u : 0u;
}

__device__ __forceinline__ void recheck_loop(const uint64_t* seg, uint32_t* sims, uint64_t seg_cap,
                                             volatile uint32_t* vcnt, volatile uint32_t* vdone,
                                             uint32_t n_epi, int rw, int nrw, const float* l32,
                                             const float* r32, int dim, float theta,
                                             uint32_t* rowcount, uint64_t start) {
  const int lane = threadIdx.x & 31;
  for (uint64_t blk = rw;; blk += nrw) {
    const uint64_t s0 = start + blk * 64;
    uint64_t n;
    for (;;) {
      n = mn<uint64_t>(*vcnt, seg_cap);
      if (n >= s0 + 64) break;
      if (*vdone == n_epi) {
        n = mn<uint64_t>(*vcnt, seg_cap);
        break;
      }
      // not latency-critical: poll rarely so the epilogue keeps the issue slots
      __nanosleep(2000);
    }
    if (s0 >= n) break;
    const uint64_t sa = s0 + lane, sb = s0 + 32 + lane;
    if (sb < n) {
      const uint64_t ua = wait_slot(seg + sa), ub = wait_slot(seg + sb);
      const uint32_t ia = (uint32_t)(ua >> 32), ja = (uint32_t)ua;
      const uint32_t ib = (uint32_t)(ub >> 32), jb = (uint32_t)ub;
      float xa, xb;
      dot_seq2_dev(l32 + (size_t)ia * dim, r32 + (size_t)ja * dim, l32 + (size_t)ib * dim,
                   r32 + (size_t)jb * dim, dim, xa, xb);
      sims[sa] = xa >= theta ? __float_as_uint(xa) : kRejected;
      sims[sb] = xb >= theta ? __float_as_uint(xb) : kRejected;
      if (xa >= theta) atomicAdd(rowcount + ia, 1u);
      if (xb >= theta) atomicAdd(rowcount + ib, 1u);
    } else if (sa < n) {
      const uint64_t ua = wait_slot(seg + sa);
      const uint32_t ia = (uint32_t)(ua >> 32), ja = (uint32_t)ua;
      const float xa = dot_seq_dev(l32 + (size_t)ia * dim, r32 + (size_t)ja * dim, dim);
      sims[sa] = xa >= theta ? __float_as_uint(xa) : kRejected;
      if (xa >= theta) atomicAdd(rowcount + ia, 1u);
    }
  }
}



}  // namespace sjb
