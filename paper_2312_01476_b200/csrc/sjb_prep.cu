// sjb_prep.cu -- prefetch-stage kernels: row L2-normalise-and-cast, the
// synthetic model fill, FNV-1a-64 hashing, and the FastText-style subword
// embedding gather.  All of them are HBM-bound; each CTA owns one 256-row
// tile, stages it in shared memory (coalesced loads), runs the per-row
// canonical arithmetic, then writes
//   * the canonical fp32 rows (bitwise equal to the reference's
//     sj_normalize_rows, _kernelcore.c:52-87), and
//   * optionally the 16-bit copy (bf16 for kpad <= 128, fp16 above) in the
//     tiled UMMA operand layout
//     (sjb_common.cuh tiled_offset), zero-padded to kpad columns.
#include "sjb_common.cuh"

#include <type_traits>

namespace sjb {

constexpr int kPrepThreads = 128;

// RN_f32(x / norm) with the correctly rounded fp64 quotient in between.
// kFast (finite norm): y = RN(1/norm) and q0 = RN(x*y) lie within 1 ulp of
// the quotient, the residual r = x - q0*norm is exact in one fma and
// RN(q0 + r*y) is the correctly rounded quotient (Markstein's theorem), i.e.
// bitwise __ddiv_rn, for every finite norm >= 1e-12 and finite float x;
// the sign goes on the float (rounding is symmetric), which keeps -0.0.
// Otherwise (inf/NaN norms) the true divide.  Callers choose kFast once per
// row (or warp), outside their element loops: a per-element test compiles to
// a divergence region around every quotient.
template <bool kFast>
__device__ __forceinline__ float quot_f32(float xf, double norm, double y) {
  const double x = (double)xf;
  if (kFast) {
    const double q0 = __dmul_rn(x, y);
    const float q = __double2float_rn(__fma_rn(__fma_rn(-q0, norm, x), y, q0));
    return __int_as_float((__float_as_int(q) & 0x7fffffff) | (__float_as_int(xf) & 0x80000000));
  }
  return __double2float_rn(__ddiv_rn(x, norm));
}

// Sequential fp64 sum of squares, repair rule, fp64 divide -- the reference's
// normalize_row (_kernelcore.c:52-70).  Operates on one smem row.  The square
// of an fp32 value is exact in fp64 (<= 48 significant bits), so the
// reference's ss + x*x (one rounding, in the add) is exactly fma(x, x, ss).
// With `err` != nullptr the same final pass also measures the row's fp16
// rounding error ||fp16(x) - x||_2 (exact squares, fp64 sum, rounded up): the
// per-row term of the filter band (sjb_common.cuh row_cutoff).
__device__ __forceinline__ int normalize_row_smem(float* row, int dim, float* err, bool bf) {
  double ss = 0.0;
  for (int d = 0; d < dim; d++) {
    double x = (double)row[d];
    ss = __fma_rn(x, x, ss);
  }
  double norm = sqrt(ss);
  int repaired = 0;
  if (norm < 1e-12) {
    row[0] = 1.0f;
    ss = 0.0;
    for (int d = 0; d < dim; d++) {
      double x = (double)row[d];
      ss = __fma_rn(x, x, ss);
    }
    norm = sqrt(ss);
    repaired = 1;
  }
  // x / norm, correctly rounded, without a full divide per element (quot_f32)
  const double y = __drcp_rn(norm);
  auto pass = [&](auto fast) {
    constexpr bool kFast = decltype(fast)::value;
    if (err == nullptr) {
      for (int d = 0; d < dim; d++) row[d] = quot_f32<kFast>(row[d], norm, y);
    } else {
      double es = 0.0;
      for (int d = 0; d < dim; d++) {
        const float x = quot_f32<kFast>(row[d], norm, y);
        row[d] = x;
        // fp16(x) - x is exact in fp32 (at most 13 significant bits, or x
        // itself when it rounds to zero), so the fp32 difference equals the
        // fp64 one
        const double e = (double)__fsub_rn(from_op16(to_op16(x, bf), bf), x);
        es = __fma_rn(e, e, es);
      }
      *err = __double2float_ru(__dmul_ru(sqrt(es), 1.0 + 1e-12));
    }
  };
  if (isfinite(norm))
    pass(std::true_type{});
  else
    pass(std::false_type{});
  return repaired;
}

// Wide rows (fewer rows per sub-tile than threads, e.g. d = 768): only the
// sum of squares must run in the reference's sequential order, one thread per
// row; the divide and the rounding-error measurement are element-parallel
// over the whole CTA.  Same bits as normalize_row_smem: the quotient is the
// same correctly rounded fp64 divide, and the error sum is our own bound
// (any summation order is within the 1 + 1e-12 factor).
constexpr int kWideRows = 32;   // rows per sub-tile handled this way (one warp of sums)

__device__ __forceinline__ double row_norm_smem(float* row, int dim, int* repaired) {
  double ss = 0.0;
  for (int d = 0; d < dim; d++) {
    const double x = (double)row[d];
    ss = __fma_rn(x, x, ss);
  }
  double norm = sqrt(ss);
  *repaired = 0;
  if (norm < 1e-12) {
    row[0] = 1.0f;
    ss = 0.0;
    for (int d = 0; d < dim; d++) {
      const double x = (double)row[d];
      ss = __fma_rn(x, x, ss);
    }
    norm = sqrt(ss);
    *repaired = 1;
  }
  return norm;
}


// Normalise the vrows (<= kWideRows) rows staged in sm; row errors to err_out
// (nullptr: not wanted).  Returns this thread's repaired-row count.
__device__ int normalize_rows_wide(float* sm, int pitch, int vrows, int dim, float* err_out,
                                   bool bf, float* inv_out = nullptr) {
  __shared__ double s_norm[kWideRows], s_y[kWideRows];
  __shared__ double s_part[kPrepThreads / 32][kWideRows];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int rep = 0;
  if (tid < vrows) {
    const double norm = row_norm_smem(sm + tid * pitch, dim, &rep);
    s_norm[tid] = norm;
    s_y[tid] = __drcp_rn(norm);
    if (inv_out != nullptr) inv_out[tid] = __double2float_rn(s_y[tid]);  // RN(1 / norm)
  }
  __syncthreads();
  const bool want = err_out != nullptr;
  for (int r = 0; r < vrows; r++) {
    const double norm = s_norm[r], y = s_y[r];
    float* row = sm + r * pitch;
    double es = 0.0;
    auto pass = [&](auto fast) {  // norm is CTA-uniform: no divergence
      constexpr bool kFast = decltype(fast)::value;
      for (int d = tid; d < dim; d += kPrepThreads) {
        const float x = quot_f32<kFast>(row[d], norm, y);
        row[d] = x;
        if (want) {
          const double e = (double)__fsub_rn(from_op16(to_op16(x, bf), bf), x);
          es = __fma_rn(e, e, es);
        }
      }
    };
    if (isfinite(norm))
      pass(std::true_type{});
    else
      pass(std::false_type{});
    if (want) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
      if (lane == 0) s_part[wid][r] = es;
    }
  }
  __syncthreads();
  if (want && tid < vrows) {
    double es = 0.0;
#pragma unroll
    for (int w = 0; w < kPrepThreads / 32; w++) es += s_part[w][tid];
    *err_out = __double2float_ru(__dmul_ru(sqrt(es), 1.0 + 1e-12));
  }
  return rep;
}

// Walks this thread's elements e = tid, tid + kPrepThreads, ... < total of a
// block of rows `dim` wide, calling f(e, r, d) with (r, d) = divmod(e, dim)
// advanced incrementally: one integer divide per thread, not per element.
template <class F>
__device__ __forceinline__ void for_each_elem(int total, int dim, F f) {
  const int qs = kPrepThreads / dim, rs = kPrepThreads - qs * dim;
  int r = (int)threadIdx.x / dim, d = (int)threadIdx.x - r * dim;
  for (int e = threadIdx.x; e < total; e += kPrepThreads) {
    f(e, r, d);
    r += qs;
    d += rs;
    if (d >= dim) {
      d -= dim;
      r++;
    }
  }
}

__device__ __forceinline__ bool aligned16(const void* p) {
  return ((uintptr_t)p & 15) == 0;
}

// Stage vrows contiguous rows of `src` (row-major, `dim` wide) into smem rows
// `pitch` floats apart; float4 loads when the rows allow it.
__device__ __forceinline__ void stage_rows(float* sm, int pitch, const float* __restrict__ src,
                                           int vrows, int dim) {
  if ((dim & 3) == 0 && aligned16(src)) {
    // batches of 8 loads in flight per thread before their stores (one load
    // at a time left wide sub-tiles latency-bound: 48 sequential round trips
    // per thread at d = 768)
    const float4* s4 = reinterpret_cast<const float4*>(src);
    const int q4 = dim >> 2, total = vrows * q4;
    constexpr int kB = 8;
    for (int e0 = threadIdx.x; e0 < total; e0 += kB * kPrepThreads) {
      float4 v[kB];
#pragma unroll
      for (int u = 0; u < kB; u++) {
        const int e = e0 + u * kPrepThreads;
        if (e < total) v[u] = __ldg(s4 + e);
      }
#pragma unroll
      for (int u = 0; u < kB; u++) {
        const int e = e0 + u * kPrepThreads;
        if (e < total) {
          const int r = e / q4, d = e - r * q4;
          float* o = sm + r * pitch + 4 * d;
          o[0] = v[u].x;
          o[1] = v[u].y;
          o[2] = v[u].z;
          o[3] = v[u].w;
        }
      }
    }
  } else {
    for_each_elem(vrows * dim, dim, [&](int e, int r, int d) { sm[r * pitch + d] = __ldg(src + e); });
  }
}

// Common tail: normalise the rows staged in `sm` (pitch floats apart) for the
// sub-tile [r0, r0 + sub) of the 256-row tile starting at row0 (`rows` valid
// rows in the whole tile), store fp32 rows and that slice of the fp16
// operand tile.
// Rounding-error outputs of a tile: row_err[i] per row, tile_err[tile] = the
// tile's maximum (accumulated in the shared `tile_max`, written by the caller).
struct ErrOut {
  float* row_err;
  unsigned* tile_max;  // smem
};

__device__ void finish_subtile(float* sm, int pitch, int r0, int sub, int rows, int dim, int kpad,
                               int64_t row0, bool normalize, float* __restrict__ out32,
                               op16_t* __restrict__ out16,
                               unsigned long long* __restrict__ repaired, ErrOut eo) {
  const int vrows = max(0, min(sub, rows - r0));  // valid rows in this sub-tile
  int rep = 0;
  const bool want = eo.row_err != nullptr;
  if (normalize && sub <= kWideRows && sub < kPrepThreads) {
    // wide rows: sequential sums per row, element-parallel divide (above)
    float e = 0.0f;
    rep = normalize_rows_wide(sm, pitch, vrows, dim, want ? &e : nullptr, op_is_bf16(kpad));
    if (want && threadIdx.x < vrows) {
      eo.row_err[row0 + r0 + threadIdx.x] = e;
      atomicMax(eo.tile_max, __float_as_uint(e));  // e >= 0: bit order = value order
    }
  } else if (normalize && threadIdx.x < vrows) {
    float e = 0.0f;
    rep = normalize_row_smem(sm + threadIdx.x * pitch, dim, want ? &e : nullptr, op_is_bf16(kpad));
    if (want) {
      eo.row_err[row0 + r0 + threadIdx.x] = e;
      atomicMax(eo.tile_max, __float_as_uint(e));  // e >= 0: bit order = value order
    }
  }
  if (normalize && repaired != nullptr) {
    rep = __reduce_add_sync(0xffffffffu, rep);
    if ((threadIdx.x & 31) == 0 && rep) atomicAdd(repaired, (unsigned long long)rep);
  }
  __syncthreads();
  if (out32 != nullptr) {
    float* dst = out32 + (row0 + r0) * dim;
    if ((dim & 3) == 0 && aligned16(dst)) {
      float4* d4 = reinterpret_cast<float4*>(dst);
      for_each_elem(vrows * (dim >> 2), dim >> 2, [&](int e, int r, int d) {
        const float* o = sm + r * pitch + 4 * d;
        d4[e] = make_float4(o[0], o[1], o[2], o[3]);
      });
    } else {
      for_each_elem(vrows * dim, dim, [&](int e, int r, int d) { dst[e] = sm[r * pitch + d]; });
    }
  }
  if (out16 != nullptr) {
    // One 16-byte chunk = 8 consecutive k of one row; consecutive threads take
    // consecutive rows of the same k-group, so each warp writes 512 B runs.
    uint4* dst = reinterpret_cast<uint4*>(out16 + (row0 / kTileRows) * (int64_t)kTileRows * kpad);
    const int nchunks = sub * (kpad / 8);
    const int lsub = 31 - __clz(sub);  // sub is a power of two
    const bool bf = op_is_bf16(kpad);
    for (int c = threadIdx.x; c < nchunks; c += kPrepThreads) {
      int g = c >> lsub, r = c & (sub - 1);
      __align__(16) op16_t v[8];
#pragma unroll
      for (int e = 0; e < 8; e++) {
        int k = g * 8 + e;
        float x = (r < vrows && k < dim) ? sm[r * pitch + k] : 0.0f;
        v[e] = to_op16(x, bf);
      }
      dst[g * kTileRows + r0 + r] = *reinterpret_cast<uint4*>(v);
    }
  }
  __syncthreads();
}

// in: n x dim fp32 row-major (or, with `gather`, a table whose row gather[i]
// is relation row i).  One CTA per 256-row operand tile, staged in sub-tiles
// of `sub` rows (sub * (dim|1) floats of smem).  The grid may cover tiles past
// n: those are written as zero operand tiles so the operand image can be padded.
__global__ void __launch_bounds__(kPrepThreads)
normalize_cast_kernel(const float* __restrict__ in, const int64_t* __restrict__ gather, int64_t n,
                      int dim, int kpad, int sub, float* __restrict__ out32,
                      op16_t* __restrict__ out16, unsigned long long* __restrict__ repaired,
                      int normalize, float* __restrict__ row_err, float* __restrict__ tile_err) {
  extern __shared__ float sm[];
  __shared__ unsigned tile_max;
  if (threadIdx.x == 0) tile_max = 0u;
  const int pitch = dim | 1;
  const int64_t row0 = (int64_t)blockIdx.x * kTileRows;
  const int rows = (int)mx<int64_t>(0, mn<int64_t>(kTileRows, n - row0));
  for (int r0 = 0; r0 < kTileRows; r0 += sub) {
    const int vrows = max(0, min(sub, rows - r0));
    if (gather == nullptr) {
      stage_rows(sm, pitch, in + (row0 + r0) * dim, vrows, dim);
    } else {  // row r of this relation is row gather[r] of `in` (lookup model)
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int r = warp; r < vrows; r += kPrepThreads / 32) {
        const float* src = in + gather[row0 + r0 + r] * (int64_t)dim;
        for (int d = lane; d < dim; d += 32) sm[r * pitch + d] = __ldg(src + d);
      }
    }
    __syncthreads();
    finish_subtile(sm, pitch, r0, sub, rows, dim, kpad, row0, normalize != 0, out32, out16,
                   repaired, ErrOut{row_err, &tile_max});
  }
  if (tile_err != nullptr && threadIdx.x == 0) tile_err[blockIdx.x] = __uint_as_float(tile_max);
}

// Pipelined normalise-and-cast (dim % 4 == 0, kpad <= 128, 16 B aligned
// input): the same bits as normalize_cast_kernel, restructured so the HBM
// stream never waits for the row-serial arithmetic.  Each warp walks 32-row
// slabs (grid-stride) with two shared buffers: while it computes slab k,
// slab k + 1 is already in flight (one 1-D bulk copy per row, lane = row,
// completing on the buffer's mbarrier).  A slab is then three passes by the
// warp, lane = row:
//   1. the reference's sequential fp64 sum of squares + repair
//      (_kernelcore.c:52-70), reading the row as float4 (row pitch = an odd
//      number of float4: conflict-free 128-bit shared loads);
//   2. the correctly rounded quotients (quot_f32, in place), the 16-bit cast
//      stored as the row's 16-byte chunks of the operand tile (a warp writes
//      one 512 B run per k-group), and the row's rounding error (exact
//      squares, fp64 sum, rounded up: the same value as the staged kernel);
//   3. the fp32 rows copied out row-major (coalesced 400 B rows).
// tile_err must be zeroed first: each slab folds its maximum in with an
// atomicMax on the bits (errors are >= 0, so bit order = value order).
constexpr int kPipeSlab = 32;
constexpr int kPipeMaxWarps = 16;

__host__ __device__ inline int pipe_pitch4(int dim) { return (dim / 4) | 1; }

// bufs = 2 (default): double-buffered, 8 warps per SM -- the next slab's
// load is in flight through the current one's arithmetic; bufs = 1: each
// warp loads its next slab after finishing the current one (16 warps)
__host__ inline int pipe_warps(int dim, int bufs, int smem_budget) {
  const int per_warp = bufs * kPipeSlab * pipe_pitch4(dim) * 16 + 16;
  return mn(kPipeMaxWarps, smem_budget / per_warp);
}

__host__ __device__ inline int pipe_smem_bytes(int dim, int bufs, int warps) {
  return warps * (bufs * kPipeSlab * pipe_pitch4(dim) * 16 + 16);
}

// Pass 2 of normalize_pipe_kernel for one row (lane = row): the correctly
// rounded quotients in place, the bf16 chunks of the operand tile and the
// row's rounding-error sum.  kFast: every lane's norm is finite, so the
// quotient is quot_f32<true> with no per-element test; otherwise
// the true divide for all lanes (the same bits where the norm is finite).
template <bool kFast>
__device__ __forceinline__ float pipe_pass2(float4* row, bool valid, int q4, int kpad, double norm,
                                            double y, uint4* dst16, int rin, bool want_err) {
  auto quot = [&](float xf) -> float { return quot_f32<kFast>(xf, norm, y); };
  float es = 0.0f;
  for (int g = 0; g < kpad / 8; g++) {
    __align__(16) float x[8];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int q = 2 * g + h;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (valid && q < q4) {
        v = row[q];
        v.x = quot(v.x);
        v.y = quot(v.y);
        v.z = quot(v.z);
        v.w = quot(v.w);
        row[q] = v;
      }
      x[4 * h + 0] = v.x;
      x[4 * h + 1] = v.y;
      x[4 * h + 2] = v.z;
      x[4 * h + 3] = v.w;
    }
    if (dst16 != nullptr) {
      // kpad <= 128: bf16 operands, converted in pairs (one F2FP per two)
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(x[2 * e], x[2 * e + 1]);
        o[e] = *reinterpret_cast<const uint32_t*>(&h);
        if (want_err) {
          // op(x) - x is exact in fp32; the squares are summed in fp32
          // rounding UP, so es bounds the exact sum from above
          const float d0 = __fsub_rn(__uint_as_float(o[e] << 16), x[2 * e]);
          const float d1 = __fsub_rn(__uint_as_float(o[e] & 0xffff0000u), x[2 * e + 1]);
          es = __fmaf_ru(d0, d0, es);
          es = __fmaf_ru(d1, d1, es);
        }
      }
      dst16[g * kTileRows + rin] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
  return es;
}

__global__ void __launch_bounds__(kPipeMaxWarps * 32, 1)
normalize_pipe_kernel(const float* __restrict__ in, int64_t n, int64_t n_slabs, int dim, int kpad,
                      int nbuf, float* out32, op16_t* __restrict__ out16,
                      unsigned long long* __restrict__ repaired, float* __restrict__ row_err,
                      unsigned* __restrict__ tile_err_bits) {
  extern __shared__ __align__(1024) uint8_t pipe_smem[];
  uint8_t* smem = pipe_smem;
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p4 = pipe_pitch4(dim), q4 = dim >> 2;
  float4* bufs = reinterpret_cast<float4*>(smem) + (size_t)warp * nbuf * kPipeSlab * p4;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem + (size_t)warps * nbuf * kPipeSlab * p4 * 16) + warp * 2;
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol = policy_evict_first();
  const int64_t nw = (int64_t)gridDim.x * warps;

  auto slab_rows = [&](int64_t slab) -> int {
    return (int)mx<int64_t>(0, mn<int64_t>(kPipeSlab, n - slab * kPipeSlab));
  };
  // q4 odd (d = 100: 25 float4): the conflict-free pitch is the row itself,
  // so a slab is one contiguous run in both global and shared memory: one
  // bulk copy in, one bulk store out (per-lane copies issue as a
  // serialised loop, and the row-by-row store loop was a quarter of the
  // kernel's stall samples)
  const bool contig = p4 == q4;
  auto issue = [&](int64_t slab, int b) {
    const int rows = slab_rows(slab);
    if (rows == 0) return;  // padding slab: nothing to load, no barrier phase
    if (lane == 0) {
      // the buffer's previous bulk store must have read it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      mbar_arrive_expect_tx(&bars[b], (uint32_t)(rows * dim * 4));
      if (contig)
        bulk_g2s(bufs + (size_t)b * kPipeSlab * p4, in + slab * kPipeSlab * (int64_t)dim,
                 (uint32_t)(rows * dim * 4), &bars[b], pol);
    }
    __syncwarp();
    if (!contig && lane < rows)
      bulk_g2s(bufs + (size_t)b * kPipeSlab * p4 + lane * p4,
               in + (slab * kPipeSlab + lane) * (int64_t)dim, (uint32_t)(dim * 4), &bars[b], pol);
  };

  uint32_t ph0 = 0, ph1 = 0;
  int b = 0;
  int64_t slab = (int64_t)blockIdx.x * warps + warp;
  if (slab < n_slabs && nbuf == 2) issue(slab, 0);
  for (; slab < n_slabs; slab += nw, b ^= (nbuf - 1)) {
    if (nbuf == 2) {
      if (slab + nw < n_slabs) issue(slab + nw, b ^ 1);
    } else {
      issue(slab, 0);
    }
    const int rows = slab_rows(slab);
    if (rows > 0) {
      if (b == 0) {
        mbar_wait(&bars[0], ph0);
        ph0 ^= 1u;
      } else {
        mbar_wait(&bars[1], ph1);
        ph1 ^= 1u;
      }
    }
    const int64_t r0 = slab * kPipeSlab;
    float4* buf = bufs + (size_t)b * kPipeSlab * p4;
    float4* row = buf + lane * p4;
    const bool valid = lane < rows;
    // ---- 1. sequential fp64 sum of squares, repair ----------------------
    int rep = 0;
    double norm = 1.0, y = 1.0;
    bool hoist = true;
    if (valid) {
      double ss = 0.0;
      for (int q = 0; q < q4; q++) {
        const float4 v = row[q];
        ss = __fma_rn((double)v.x, (double)v.x, ss);
        ss = __fma_rn((double)v.y, (double)v.y, ss);
        ss = __fma_rn((double)v.z, (double)v.z, ss);
        ss = __fma_rn((double)v.w, (double)v.w, ss);
      }
      norm = sqrt(ss);
      if (norm < 1e-12) {
        float4 v0 = row[0];
        v0.x = 1.0f;
        row[0] = v0;
        ss = 0.0;
        for (int q = 0; q < q4; q++) {
          const float4 v = row[q];
          ss = __fma_rn((double)v.x, (double)v.x, ss);
          ss = __fma_rn((double)v.y, (double)v.y, ss);
          ss = __fma_rn((double)v.z, (double)v.z, ss);
          ss = __fma_rn((double)v.w, (double)v.w, ss);
        }
        norm = sqrt(ss);
        rep = 1;
      }
      hoist = isfinite(norm);
      y = __drcp_rn(norm);
    }
    // ---- 2. quotients (in place), operand chunks, rounding error --------
    const int64_t tile = r0 / kTileRows;
    const int rin = (int)(r0 - tile * kTileRows) + lane;
    uint4* dst16 = out16 != nullptr
                       ? reinterpret_cast<uint4*>(out16 + tile * (int64_t)kTileRows * kpad)
                       : nullptr;
    // warp-uniform choice: the per-element loop carries no branch (a per-lane
    // hoist test around every quotient compiled to a divergence region per
    // element and doubled the kernel's issue count)
    const float es = __all_sync(0xffffffffu, hoist)
                         ? pipe_pass2<true>(row, valid, q4, kpad, norm, y, dst16, rin, row_err != nullptr)
                         : pipe_pass2<false>(row, valid, q4, kpad, norm, y, dst16, rin, row_err != nullptr);
    __syncwarp();
    // ---- 3. fp32 rows out, errors, counters -----------------------------
    if (out32 != nullptr && contig) {
      if (rows > 0) {
        // pass 2's shared writes become visible to the async proxy, then
        // one bulk store (completion awaited before the buffer's next load)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0)
          asm volatile(
              "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
              "cp.async.bulk.commit_group;" ::"l"(out32 + r0 * (int64_t)dim),
              "r"(smem_u32(buf)), "r"((uint32_t)(rows * dim * 4))
              : "memory");
      }
    } else if (out32 != nullptr) {
      float4* o4 = reinterpret_cast<float4*>(out32 + r0 * (int64_t)dim);
      for (int r = 0; r < rows; r++)
        for (int q = lane; q < q4; q += 32) o4[r * q4 + q] = buf[r * p4 + q];
    }
    if (row_err != nullptr && dst16 != nullptr && rows > 0) {
      float e = 0.0f;
      if (valid) {
        e = __fmul_ru(__fsqrt_ru(es), 1.0f + 1e-6f);
        row_err[r0 + lane] = e;
      }
      const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(e));
      if (lane == 0 && tile_err_bits != nullptr) atomicMax(tile_err_bits + tile, m);
    }
    if (repaired != nullptr) {
      rep = __reduce_add_sync(0xffffffffu, rep);
      if (lane == 0 && rep) atomicAdd(repaired, (unsigned long long)rep);
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// bf16 relations for the raw-operand wide filter (BASELINE cfg4: d = 768
// bf16 inputs).  The operand image holds the RAW bf16 rows (exact: the
// tensor-core products of bf16 values are exact, so the filter's error is
// only fp32 accumulation), the fp32 outputs are the canonical normalised rows
// (bitwise sj_normalize_rows of the rows' fp32 values, which the bf16 values
// are exactly), and inv_norm[i] = RN(1 / ||x_i||) for the epilogue's
// normalise-after-GEMM.  A repaired (near-zero) row gets component 0 := 1 in
// its raw image too, like the reference's row.  One CTA per 256-row tile,
// 32-row sub-tiles (sequential fp64 sums one thread per row, element-parallel
// divide: normalize_rows_wide).  Rows >= n (tile padding) get zero operands
// and inv_norm 0.
__global__ void __launch_bounds__(kPrepThreads)
prepare_bf16_kernel(const uint16_t* __restrict__ in, int64_t n, int dim, int kpad,
                    float* __restrict__ out32, op16_t* __restrict__ out16,
                    float* __restrict__ inv_norm, unsigned long long* __restrict__ repaired) {
  extern __shared__ float sm[];
  __shared__ float s_inv[kWideRows];
  const int pitch = dim | 1;
  const int64_t row0 = (int64_t)blockIdx.x * kTileRows;
  const int rows = (int)mx<int64_t>(0, mn<int64_t>(kTileRows, n - row0));
  op16_t* tile16 = out16 + (row0 / kTileRows) * (int64_t)kTileRows * kpad;
  const int ngrp = kpad / 8;
  for (int r0 = 0; r0 < kTileRows; r0 += kWideRows) {
    const int vrows = max(0, min(kWideRows, rows - r0));
    // raw operand chunks (8 k of one row: 16 B) straight from the input, and
    // the rows' fp32 values into shared memory
    for (int c = threadIdx.x; c < kWideRows * ngrp; c += kPrepThreads) {
      const int g = c / kWideRows, r = c - g * kWideRows;
      __align__(16) op16_t v[8];
      if (r < vrows) {
        const uint16_t* src = in + (row0 + r0 + r) * (int64_t)dim + g * 8;
        if (g * 8 + 8 <= dim && ((dim & 7) == 0)) {
          *reinterpret_cast<uint4*>(v) = __ldg(reinterpret_cast<const uint4*>(src));
        } else {
#pragma unroll
          for (int e = 0; e < 8; e++) v[e] = g * 8 + e < dim ? src[e] : (op16_t)0;
        }
#pragma unroll
        for (int e = 0; e < 8; e++)
          if (g * 8 + e < dim)
            sm[r * pitch + g * 8 + e] = __bfloat162float(__ushort_as_bfloat16(v[e]));
      } else {
#pragma unroll
        for (int e = 0; e < 8; e++) v[e] = 0;
      }
      reinterpret_cast<uint4*>(tile16)[g * kTileRows + r0 + r] = *reinterpret_cast<uint4*>(v);
    }
    __syncthreads();
    int rep = normalize_rows_wide(sm, pitch, vrows, dim, nullptr, true, s_inv);
    if (threadIdx.x < kWideRows)
      inv_norm[row0 + r0 + threadIdx.x] = threadIdx.x < vrows ? s_inv[threadIdx.x] : 0.0f;
    if (rep && threadIdx.x < vrows)   // the reference's repaired row has x[0] = 1
      tile16[(r0 + threadIdx.x) * 8] = (op16_t)0x3F80;   // bf16(1.0): k-group 0, element 0
    if (repaired != nullptr) {
      rep = __reduce_add_sync(0xffffffffu, rep);
      if ((threadIdx.x & 31) == 0 && rep) atomicAdd(repaired, (unsigned long long)rep);
    }
    __syncthreads();
    float* dst = out32 + (row0 + r0) * (int64_t)dim;
    for_each_elem(vrows * dim, dim, [&](int e, int r, int d) { dst[e] = sm[r * pitch + d]; });
    __syncthreads();
  }
}

// Synthetic model (_kernelcore.c:42-50, 72-80): stream seed per row, element
// d = splitmix64 output d+1 mapped to fp64 [-1,1), truncated to fp32, then the
// row is normalised.  Element-parallel generation, row-serial normalisation.
__device__ __forceinline__ float splitmix_elem(uint64_t seed, int d) {
  uint64_t z = seed + (uint64_t)(d + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z = z ^ (z >> 31);
  double v = __dsub_rn(__dmul_rn(__dmul_rn((double)z, 0x1p-64), 2.0), 1.0);
  return __double2float_rn(v);
}

__global__ void __launch_bounds__(kPrepThreads)
synthetic_fill_kernel(const uint64_t* __restrict__ seeds, int64_t n, int dim, int kpad, int sub,
                      float* __restrict__ out32, op16_t* __restrict__ out16,
                      float* __restrict__ row_err, float* __restrict__ tile_err) {
  extern __shared__ float sm[];
  __shared__ unsigned tile_max;
  if (threadIdx.x == 0) tile_max = 0u;
  const int pitch = dim | 1;
  const int64_t row0 = (int64_t)blockIdx.x * kTileRows;
  const int rows = (int)mx<int64_t>(0, mn<int64_t>(kTileRows, n - row0));
  for (int r0 = 0; r0 < kTileRows; r0 += sub) {
    const int vrows = max(0, min(sub, rows - r0));
    for_each_elem(vrows * dim, dim, [&](int, int r, int d) {
      sm[r * pitch + d] = splitmix_elem(seeds[row0 + r0 + r], d);
    });
    __syncthreads();
    // synthetic vectors are normalised as part of the model (embedding.py:79)
    finish_subtile(sm, pitch, r0, sub, rows, dim, kpad, row0, true, out32, out16, nullptr,
                   ErrOut{row_err, &tile_max});
  }
  if (tile_err != nullptr && threadIdx.x == 0) tile_err[blockIdx.x] = __uint_as_float(tile_max);
}

// FNV-1a-64 (_kernelcore.c:33-40) of packed tokens, XOR a 64-bit seed
// (SyntheticModel._stream_seed, embedding.py:87-88).
__global__ void fnv1a64_kernel(const uint8_t* __restrict__ bytes, const int64_t* __restrict__ offs,
                               int64_t n, uint64_t xor_seed, uint64_t* __restrict__ out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t i = offs[t]; i < offs[t + 1]; i++) {
    h ^= (uint64_t)bytes[i];
    h *= 0x100000001b3ULL;
  }
  out[t] = h ^ xor_seed;
}

// ------------------------------------------------------------------------
// Subword (FastText-style) model, cfg3.  Builder-pinned spec (the reference
// has no subword model; restated in oracle/sj_oracle.c):
// items = [word row] + [every n-gram of '<' w '>' for n = minn..maxn, by n then
// start]; bucket = fnv1a64(bytes) mod n_buckets; row = (sum of item rows in
// item order, fp32) / (float)count.  One warp per token; lanes own columns,
// so each column is accumulated sequentially in item order (bit-exact with
// the oracle) and every gathered row is read as coalesced 128 B segments.
__device__ __forceinline__ uint8_t marked_byte(const uint8_t* w, int len, int k) {
  return k == 0 ? (uint8_t)'<' : (k == len + 1 ? (uint8_t)'>' : w[k - 1]);
}

// Sum the table rows of a batch of nb items (bucket of item q in lane q) into
// this lane's columns lane + 32k (k < C), in item order (fp32, exactly the
// sequential sum), with 8 items' loads issued before their adds.
#ifndef SJB_SUBWORD_KU
#define SJB_SUBWORD_KU 8
#endif
template <int C>
__device__ __forceinline__ void gather_items(float* acc, const float* __restrict__ table,
                                             uint64_t bucket, int nb, int dim, int lane) {
  constexpr int kU = SJB_SUBWORD_KU;
  for (int q0 = 0; q0 < nb; q0 += kU) {
    float v[kU][C];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const uint64_t bq = __shfl_sync(0xffffffffu, bucket, (q0 + u) & 31);
      const float* src = table + bq * (uint64_t)dim;
#pragma unroll
      for (int k = 0; k < C; k++)
        v[u][k] = (q0 + u < nb && lane + 32 * k < dim) ? __ldg(src + lane + 32 * k) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kU; u++)
      if (q0 + u < nb) {
#pragma unroll
        for (int k = 0; k < C; k++) acc[k] = __fadd_rn(acc[k], v[u][k]);
      }
  }
}

__global__ void __launch_bounds__(kPrepThreads, 8)  // 8 CTAs/SM: the gather is latency-bound
subword_embed_kernel(const uint8_t* __restrict__ bytes, const int64_t* __restrict__ offs,
                     int64_t n, const float* __restrict__ table, int64_t n_buckets, int dim,
                     int kpad, int sub, int minn, int maxn, int normalize,
                     float* __restrict__ out32, op16_t* __restrict__ out16,
                     unsigned long long* __restrict__ repaired, float* __restrict__ row_err,
                     float* __restrict__ tile_err) {
  extern __shared__ float sm[];
  __shared__ unsigned tile_max;
  if (threadIdx.x == 0) tile_max = 0u;
  const int pitch = dim | 1;
  const int64_t row0 = (int64_t)blockIdx.x * kTileRows;
  const int rows = (int)mx<int64_t>(0, mn<int64_t>(kTileRows, n - row0));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r0 = 0; r0 < kTileRows; r0 += sub) {
    const int vrows = max(0, min(sub, rows - r0));
    for (int r = warp; r < vrows; r += kPrepThreads / 32) {
      const int64_t t = row0 + r0 + r;
      const uint8_t* w = bytes + offs[t];
      const int len = (int)(offs[t + 1] - offs[t]);
      const int ml = len + 2;
      int n_items = 1;
      for (int g = minn; g <= maxn; g++) n_items += max(0, ml - g + 1);
      float* row = sm + r * pitch;
      const int ncol = (dim + 31) / 32;
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      if (ncol > 4)
        for (int d = lane; d < dim; d += 32) row[d] = 0.0f;
      for (int b0 = 0; b0 < n_items; b0 += 32) {
        // lane computes the bucket of item b0 + lane
        const int item = b0 + lane;
        uint64_t bucket = 0;
        if (item < n_items) {
          uint64_t h = 0xcbf29ce484222325ULL;
          if (item == 0) {
            for (int k = 0; k < len; k++) {
              h ^= (uint64_t)w[k];
              h *= 0x100000001b3ULL;
            }
          } else {
            int rem = item - 1, g = minn;
            while (rem >= max(0, ml - g + 1)) {
              rem -= max(0, ml - g + 1);
              g++;
            }
            for (int k = rem; k < rem + g; k++) {
              h ^= (uint64_t)marked_byte(w, len, k);
              h *= 0x100000001b3ULL;
            }
          }
          bucket = h % (uint64_t)n_buckets;
        }
        const int nb = min(32, n_items - b0);
        switch (ncol) {  // register accumulation, item loads in flight together
          case 1: gather_items<1>(acc, table, bucket, nb, dim, lane); break;
          case 2: gather_items<2>(acc, table, bucket, nb, dim, lane); break;
          case 3: gather_items<3>(acc, table, bucket, nb, dim, lane); break;
          case 4: gather_items<4>(acc, table, bucket, nb, dim, lane); break;
          default:
            for (int q = 0; q < nb; q++) {
              const uint64_t bq = __shfl_sync(0xffffffffu, bucket, q);
              const float* src = table + bq * (uint64_t)dim;
              for (int d = lane; d < dim; d += 32) row[d] = __fadd_rn(row[d], __ldg(src + d));
            }
        }
      }
      const float c = (float)n_items;
      if (ncol <= 4) {
#pragma unroll
        for (int k = 0; k < 4; k++)
          if (k < ncol && lane + 32 * k < dim) row[lane + 32 * k] = __fdiv_rn(acc[k], c);
      } else {
        for (int d = lane; d < dim; d += 32) row[d] = __fdiv_rn(row[d], c);
      }
    }
    __syncthreads();
    finish_subtile(sm, pitch, r0, sub, rows, dim, kpad, row0, normalize != 0, out32, out16,
                   repaired, ErrOut{row_err, &tile_max});
  }
  if (tile_err != nullptr && threadIdx.x == 0) tile_err[blockIdx.x] = __uint_as_float(tile_max);
}

// Gather-only subword embedding (dim % 4 == 0, dim <= 128 * V): one warp per
// string, grid-stride over the strings.  Lane q hashes item q of the batch;
// lane l owns the float4 columns l + 32 v (v < V), so every item row is read
// with 16-byte loads (a d = 100 row is 25 float4 = 25 lanes) and KU items'
// loads are in flight before their adds, which run in item order per column
// (bit-exact with the sequential fp32 sum).  Writes the mean rows (fp32,
// row-major, coalesced float4 stores); normalisation and the operand image
// are a separate normalize_cast pass over these rows (from L2 at cfg3
// sizes), so this kernel is nothing but the HBM gather.
__device__ __forceinline__ uint64_t mod_u64(uint64_t h, uint64_t d, uint64_t magic) {
  // magic = floor((2^64 - 1) / d): q is floor(h / d) or at most 2 below
  uint64_t r = h - __umul64hi(h, magic) * d;
  while (r >= d) r -= d;
  return r;
}

__device__ __forceinline__ uint64_t subword_item_bucket(const uint8_t* __restrict__ w, int len,
                                                        int item, int minn, uint64_t nb,
                                                        uint64_t magic) {
  uint64_t h = 0xcbf29ce484222325ULL;
  if (item == 0) {
    for (int k = 0; k < len; k++) {
      h ^= (uint64_t)w[k];
      h *= 0x100000001b3ULL;
    }
  } else {
    const int ml = len + 2;
    int rem = item - 1, g = minn;
    while (rem >= max(0, ml - g + 1)) {
      rem -= max(0, ml - g + 1);
      g++;
    }
    for (int k = rem; k < rem + g; k++) {
      h ^= (uint64_t)marked_byte(w, len, k);
      h *= 0x100000001b3ULL;
    }
  }
  return mod_u64(h, nb, magic);
}

constexpr int kGatherThreads = 256;

template <int V, int KU, int MINB>
__global__ void __launch_bounds__(kGatherThreads, MINB)
subword_gather_kernel(const uint8_t* __restrict__ bytes, const int64_t* __restrict__ offs,
                      int64_t n, const float* __restrict__ table, uint64_t n_buckets,
                      uint64_t magic, int dim, int minn, int maxn, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * kGatherThreads) >> 5;
  const int q4 = dim >> 2;
  const float4* __restrict__ t4 = reinterpret_cast<const float4*>(table);
  float4* __restrict__ o4 = reinterpret_cast<float4*>(out);
  for (int64_t t = ((int64_t)blockIdx.x * kGatherThreads + threadIdx.x) >> 5; t < n; t += nwarps) {
    const int64_t b = offs[t];
    const int len = (int)(offs[t + 1] - b);
    const uint8_t* w = bytes + b;
    const int ml = len + 2;
    int n_items = 1;
    for (int g = minn; g <= maxn; g++) n_items += max(0, ml - g + 1);
    float4 acc[V];
#pragma unroll
    for (int v = 0; v < V; v++) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int b0 = 0; b0 < n_items; b0 += 32) {
      const int item = b0 + lane;
      const uint64_t bucket =
          item < n_items ? subword_item_bucket(w, len, item, minn, n_buckets, magic) : 0;
      const int nb = min(32, n_items - b0);
      for (int q0 = 0; q0 < nb; q0 += KU) {
        float4 val[KU][V];
#pragma unroll
        for (int u = 0; u < KU; u++) {
          const uint64_t bq = __shfl_sync(0xffffffffu, bucket, (q0 + u) & 31);
          const float4* src = t4 + bq * (uint64_t)q4;
#pragma unroll
          for (int v = 0; v < V; v++) {
            const int c = lane + 32 * v;
            val[u][v] = (q0 + u < nb && c < q4) ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < KU; u++)
          if (q0 + u < nb) {
#pragma unroll
            for (int v = 0; v < V; v++) {
              acc[v].x = __fadd_rn(acc[v].x, val[u][v].x);
              acc[v].y = __fadd_rn(acc[v].y, val[u][v].y);
              acc[v].z = __fadd_rn(acc[v].z, val[u][v].z);
              acc[v].w = __fadd_rn(acc[v].w, val[u][v].w);
            }
          }
      }
    }
    const float cnt = (float)n_items;
#pragma unroll
    for (int v = 0; v < V; v++) {
      const int c = lane + 32 * v;
      if (c < q4)
        o4[t * q4 + c] = make_float4(__fdiv_rn(acc[v].x, cnt), __fdiv_rn(acc[v].y, cnt),
                                     __fdiv_rn(acc[v].z, cnt), __fdiv_rn(acc[v].w, cnt));
    }
  }
}

// Row L2 norms in fp64, returned as fp32 (sj_row_norms, _kernelcore.c:89-99).
__global__ void row_norms_kernel(const float* __restrict__ m, int64_t n, int dim,
                                 float* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* row = m + i * dim;
  double ss = 0.0;
  for (int d = 0; d < dim; d++) {
    double x = (double)row[d];
    ss = __fma_rn(x, x, ss);
  }
  out[i] = __double2float_rn(sqrt(ss));
}

}  // namespace sjb
