// sjb_post.cu -- everything after the tensor-core filter:
//
//   (the canonical recheck runs inside the filter kernel, sjb_join.cu)
//   row scan   exclusive prefix sum of per-row match counts
//   scatter    bucket kept pairs by left row (counting sort)
//   segsort    sort each left row's bucket by right offset and write the
//              MatchSet columns (u64 lefts, u64 rights, f32 sims) -- the
//              canonical (left, right) order of canonicalize (core.py:196-213).
//
// plus the dense kernels behind the reference backend API:
//   tile_dot   canonical dense tile (sj_tile_dot, _kernelcore.c:300-323)
//   dots_vm    sj_dots_vm (_kernelcore.c:108-111)
//   scan_hits  row-major threshold scan of a dense buffer (_kernelcore.c:300-323)
#include "sjb_common.cuh"

namespace sjb {

// ----------------------------------------------------------- prefix scan
// Three-phase exclusive scan of u32 counts into u64 offsets (n+1 entries).
constexpr int kScanThreads = 1024;
constexpr int kScanPerThread = 4;
constexpr int kScanBlock = kScanThreads * kScanPerThread;

__device__ __forceinline__ uint64_t block_excl_scan(uint64_t x, uint64_t* warp_sums,
                                                    uint64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint64_t w = lane < nw ? warp_sums[lane] : 0;
    uint64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < nw) warp_sums[lane] = wi - w;
    if (lane == nw - 1) *total = wi;
  }
  __syncthreads();
  const uint64_t r = warp_sums[warp] + incl - x;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads)
scan_reduce_kernel(const uint32_t* __restrict__ in, int64_t n, uint64_t* __restrict__ block_sums) {
  __shared__ uint64_t ws[32];
  __shared__ uint64_t tot;
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + threadIdx.x * kScanPerThread;
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; k++)
    if (base + k < n) s += in[base + k];
  block_excl_scan(s, ws, &tot);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

// Single block: exclusive scan of the block sums in place (nb <= 4096).
__global__ void __launch_bounds__(kScanThreads)
scan_blocks_kernel(uint64_t* __restrict__ block_sums, int64_t nb, uint64_t* __restrict__ grand) {
  __shared__ uint64_t ws[32];
  __shared__ uint64_t tot;
  const int64_t base = threadIdx.x * kScanPerThread;
  uint64_t v[kScanPerThread];
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; k++) {
    v[k] = base + k < nb ? block_sums[base + k] : 0;
    s += v[k];
  }
  uint64_t off = block_excl_scan(s, ws, &tot);
#pragma unroll
  for (int k = 0; k < kScanPerThread; k++) {
    if (base + k < nb) block_sums[base + k] = off;
    off += v[k];
  }
  if (threadIdx.x == 0) *grand = tot;
}

__global__ void __launch_bounds__(kScanThreads)
scan_down_kernel(const uint32_t* __restrict__ in, int64_t n, const uint64_t* __restrict__ block_sums,
                 const uint64_t* __restrict__ grand, uint64_t* __restrict__ out,
                 uint64_t* __restrict__ out_copy) {
  __shared__ uint64_t ws[32];
  __shared__ uint64_t tot;
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + threadIdx.x * kScanPerThread;
  uint32_t v[kScanPerThread];
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; k++) {
    v[k] = base + k < n ? in[base + k] : 0u;
    s += v[k];
  }
  uint64_t off = block_excl_scan(s, ws, &tot) + block_sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanPerThread; k++) {
    if (base + k < n) {
      out[base + k] = off;
      if (out_copy) out_copy[base + k] = off;
    }
    off += v[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[n] = *grand;
    if (out_copy) out_copy[n] = *grand;
  }
}

// ------------------------------------------------------------- scatter
// Sort key = (right offset << 32) | sim bits: unique per row because right
// offsets are unique within a row.  gate[1] == 0 (matches exceed the output
// capacity) turns scatter and sort into no-ops; the host retries.
// ---------------------------------------------- dense (row-grouped) recheck
// For dense joins (deferred mode) the candidates are first grouped by left
// row, so the canonical recheck reads each R row from L1 for all of that
// row's candidates and only the S rows come from L2:
//   count_rows -> scan -> group_rows -> recheck_grouped -> scan -> compact
// Segment kernels run on a 2-D grid: blockIdx.y = segment.
// (+ sig != nullptr: each row's smallest right offset, sig preset to ~0)
__global__ void count_rows_kernel(const uint64_t* __restrict__ cand, uint64_t seg_cap,
                                  const unsigned long long* __restrict__ cta_count,
                                  uint32_t* __restrict__ rowcount, uint32_t* __restrict__ sig) {
  const unsigned long long cc = cta_count[blockIdx.y];
  if (cc > seg_cap) return;  // saturated segment: the join is retried with room
  const uint64_t* seg = cand + (uint64_t)blockIdx.y * seg_cap;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cc;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = seg[k];
    atomicAdd(rowcount + (uint32_t)(u >> 32), 1u);
    if (sig) atomicMin(sig + (uint32_t)(u >> 32), (uint32_t)u);
  }
}

__global__ void group_rows_kernel(const uint64_t* __restrict__ cand, uint64_t seg_cap,
                                  const unsigned long long* __restrict__ cta_count,
                                  unsigned long long* __restrict__ cursor,
                                  uint64_t* __restrict__ grouped) {
  const unsigned long long cc = cta_count[blockIdx.y];
  if (cc > seg_cap) return;
  const uint64_t* seg = cand + (uint64_t)blockIdx.y * seg_cap;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cc;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = seg[k];
    grouped[atomicAdd(cursor + (uint32_t)(u >> 32), 1ull)] = u;
  }
}

// The same two passes with per-chunk aggregation: a CTA takes 2048
// consecutive candidates of one segment.  A filter CTA appends its work
// items (256-row R blocks) one after another, so a chunk's rows nearly always
// lie within one or two blocks: when they span < kAggSpan rows, counts (and
// signature minima) are taken in shared memory and folded into the global
// arrays with one atomic per distinct row, and the grouping reserves each
// row's run of the chunk with one returning atomic (local ranks from the
// shared counters).  Wider chunks fall back to per-candidate atomics.
#ifndef SJB_AGG_THREADS
#define SJB_AGG_THREADS 256
#endif
constexpr int kAggThreads = SJB_AGG_THREADS;
#ifndef SJB_AGG_PER
#define SJB_AGG_PER 8
#endif
constexpr int kAggPer = SJB_AGG_PER;
constexpr int kAggChunk = kAggThreads * kAggPer;
constexpr int kAggSpan = 2048;

__device__ __forceinline__ void agg_row_range(const uint64_t (&u)[kAggPer], int n, uint32_t* s_mm,
                                              uint32_t& rmin, uint32_t& rmax) {
  uint32_t lo = ~0u, hi = 0u;
#pragma unroll
  for (int e = 0; e < kAggPer; e++) {
    const int k = threadIdx.x + kAggThreads * e;
    if (k < n) {
      const uint32_t r = (uint32_t)(u[e] >> 32);
      lo = min(lo, r);
      hi = max(hi, r);
    }
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&s_mm[0], lo);
    atomicMax(&s_mm[1], hi);
  }
  __syncthreads();
  rmin = s_mm[0];
  rmax = s_mm[1];
}

__global__ void __launch_bounds__(kAggThreads)
count_rows_agg_kernel(const uint64_t* __restrict__ cand, uint64_t seg_cap,
                      const unsigned long long* __restrict__ cta_count,
                      uint32_t* __restrict__ rowcount, uint32_t* __restrict__ sig) {
  __shared__ uint32_t hcnt[kAggSpan], hmin[kAggSpan];
  __shared__ uint32_t s_mm[2];
  const unsigned long long cc = cta_count[blockIdx.y];
  if (cc > seg_cap) return;  // saturated segment: the join is retried with room
  const uint64_t* seg = cand + (uint64_t)blockIdx.y * seg_cap;
  for (uint64_t k0 = (uint64_t)blockIdx.x * kAggChunk; k0 < cc;
       k0 += (uint64_t)gridDim.x * kAggChunk) {
    const int n = (int)mn<uint64_t>(kAggChunk, cc - k0);
    uint64_t u[kAggPer];
#pragma unroll
    for (int e = 0; e < kAggPer; e++) {
      const int k = threadIdx.x + kAggThreads * e;
      u[e] = k < n ? seg[k0 + k] : 0ull;
    }
    if (threadIdx.x == 0) {
      s_mm[0] = ~0u;
      s_mm[1] = 0u;
    }
    __syncthreads();
    uint32_t rmin, rmax;
    agg_row_range(u, n, s_mm, rmin, rmax);
    const uint32_t span = rmax - rmin + 1;
    if (span <= (uint32_t)kAggSpan) {
      for (uint32_t r = threadIdx.x; r < span; r += kAggThreads) {
        hcnt[r] = 0u;
        hmin[r] = ~0u;
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < kAggPer; e++) {
        const int k = threadIdx.x + kAggThreads * e;
        if (k < n) {
          const uint32_t r = (uint32_t)(u[e] >> 32) - rmin;
          atomicAdd(&hcnt[r], 1u);
          atomicMin(&hmin[r], (uint32_t)u[e]);
        }
      }
      __syncthreads();
      for (uint32_t r = threadIdx.x; r < span; r += kAggThreads) {
        const uint32_t c = hcnt[r];
        if (c) {
          atomicAdd(rowcount + rmin + r, c);
          atomicMin(sig + rmin + r, hmin[r]);
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < kAggPer; e++) {
        const int k = threadIdx.x + kAggThreads * e;
        if (k < n) {
          atomicAdd(rowcount + (uint32_t)(u[e] >> 32), 1u);
          atomicMin(sig + (uint32_t)(u[e] >> 32), (uint32_t)u[e]);
        }
      }
    }
    __syncthreads();
  }
}

// OutT = uint32_t: only the right offset is stored (the dense recheck's
// grouped array: rows at cursor-given offsets, the row known from them)
template <class OutT>
__global__ void __launch_bounds__(kAggThreads)
group_rows_agg_kernel(const uint64_t* __restrict__ cand, uint64_t seg_cap,
                      const unsigned long long* __restrict__ cta_count,
                      unsigned long long* __restrict__ cursor, OutT* __restrict__ grouped) {
  __shared__ uint32_t hcnt[kAggSpan];
  __shared__ unsigned long long hbase[kAggSpan];
  __shared__ uint32_t s_mm[2];
  const unsigned long long cc = cta_count[blockIdx.y];
  if (cc > seg_cap) return;
  const uint64_t* seg = cand + (uint64_t)blockIdx.y * seg_cap;
  for (uint64_t k0 = (uint64_t)blockIdx.x * kAggChunk; k0 < cc;
       k0 += (uint64_t)gridDim.x * kAggChunk) {
    const int n = (int)mn<uint64_t>(kAggChunk, cc - k0);
    uint64_t u[kAggPer];
#pragma unroll
    for (int e = 0; e < kAggPer; e++) {
      const int k = threadIdx.x + kAggThreads * e;
      u[e] = k < n ? seg[k0 + k] : 0ull;
    }
    if (threadIdx.x == 0) {
      s_mm[0] = ~0u;
      s_mm[1] = 0u;
    }
    __syncthreads();
    uint32_t rmin, rmax;
    agg_row_range(u, n, s_mm, rmin, rmax);
    const uint32_t span = rmax - rmin + 1;
    if (span <= (uint32_t)kAggSpan) {
      for (uint32_t r = threadIdx.x; r < span; r += kAggThreads) hcnt[r] = 0u;
      __syncthreads();
      uint32_t rank[kAggPer];
#pragma unroll
      for (int e = 0; e < kAggPer; e++) {
        const int k = threadIdx.x + kAggThreads * e;
        rank[e] = k < n ? atomicAdd(&hcnt[(uint32_t)(u[e] >> 32) - rmin], 1u) : 0u;
      }
      __syncthreads();
      for (uint32_t r = threadIdx.x; r < span; r += kAggThreads) {
        const uint32_t c = hcnt[r];
        if (c) hbase[r] = atomicAdd(cursor + rmin + r, (unsigned long long)c);
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < kAggPer; e++) {
        const int k = threadIdx.x + kAggThreads * e;
        if (k < n) grouped[hbase[(uint32_t)(u[e] >> 32) - rmin] + rank[e]] = (OutT)u[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < kAggPer; e++) {
        const int k = threadIdx.x + kAggThreads * e;
        if (k < n) grouped[atomicAdd(cursor + (uint32_t)(u[e] >> 32), 1ull)] = (OutT)u[e];
      }
    }
    __syncthreads();
  }
}

// grouped[0 .. *total) holds (i << 32 | j) grouped by i: consecutive threads
// share the R row (L1), S rows come from L2 (the sequential chain of
// dot_seq_dev = sj_dot_seq).  Staging the warp's S rows in shared memory was
// measured slower (7.4 -> 14.5 ms at cfg5).
__global__ void __launch_bounds__(256)
recheck_grouped_kernel(const uint64_t* __restrict__ grouped, const uint64_t* __restrict__ total,
                       const float* __restrict__ l32, const float* __restrict__ r32, int dim,
                       float theta, uint32_t* __restrict__ sims_bits,
                       uint32_t* __restrict__ rowcount) {
  const uint64_t n = *total;
  // R rows stream through once per row group (evict first); S rows are
  // re-read by every row of their cluster (keep them in L2)
  const uint64_t pol_r = policy_evict_first(), pol_s = policy_evict_last();
  const bool vec = (dim & 3) == 0 && ((reinterpret_cast<uintptr_t>(l32) |
                                       reinterpret_cast<uintptr_t>(r32)) & 15) == 0;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = grouped[k];
    const uint32_t gi = (uint32_t)(u >> 32), gj = (uint32_t)u;
    const float* a = l32 + (size_t)gi * dim;
    const float* b = r32 + (size_t)gj * dim;
    float x = 0.0f;
    if (vec) {
      // S rows through 32-byte loads (one whole sector per lane: the kernel
      // is bound by L1 tag lookups); a row 16 bytes off a sector boundary
      // takes its first 4 elements as a 16-byte load.  Same d order.
      int d = 0;
      if (reinterpret_cast<uintptr_t>(b) & 16) {
        const float4 p = ldg4_hint(a, pol_r), q = ldg4_hint(b, pol_s);
        x = __fmaf_rn(p.x, q.x, x);
        x = __fmaf_rn(p.y, q.y, x);
        x = __fmaf_rn(p.z, q.z, x);
        x = __fmaf_rn(p.w, q.w, x);
        d = 4;
      }
#pragma unroll 3
      for (; d + 8 <= dim; d += 8) {
        const f8 q = ldg8_hint(b + d, pol_s);
        const float4 p0 = ldg4_hint(a + d, pol_r), p1 = ldg4_hint(a + d + 4, pol_r);
        x = __fmaf_rn(p0.x, q.v[0], x);
        x = __fmaf_rn(p0.y, q.v[1], x);
        x = __fmaf_rn(p0.z, q.v[2], x);
        x = __fmaf_rn(p0.w, q.v[3], x);
        x = __fmaf_rn(p1.x, q.v[4], x);
        x = __fmaf_rn(p1.y, q.v[5], x);
        x = __fmaf_rn(p1.z, q.v[6], x);
        x = __fmaf_rn(p1.w, q.v[7], x);
      }
      if (d < dim) {   // dim % 8 == 4 tail
        const float4 p = ldg4_hint(a + d, pol_r), q = ldg4_hint(b + d, pol_s);
        x = __fmaf_rn(p.x, q.x, x);
        x = __fmaf_rn(p.y, q.y, x);
        x = __fmaf_rn(p.z, q.z, x);
        x = __fmaf_rn(p.w, q.w, x);
      }
    } else {
      x = dot_seq_dev(a, b, dim);
    }
    const bool ok = x >= theta;
    sims_bits[k] = ok ? __float_as_uint(x) : kRejected;
    if (ok) atomicAdd(rowcount + gi, 1u);
  }
}

// ------------------------------------ dense recheck, sorted rows, TMA rows
// The row-grouped recheck above gathers S rows with per-lane loads: every
// load instruction touches 32 lines, so the kernel is bound by L1 wavefronts
// (68% of peak, 6.3 ms at cfg5 theta = 0.4), and the row sort, the compaction
// and the keys round trip after it cost 3.8 ms more.  Here one warp owns one
// left row at a time (rows handed out by a global counter):
//  * a row of n <= kRowSortCap candidates has its right offsets sorted
//    ascending in registers (u32 bitonic) and parked in the warp's shared
//    list, so the recheck already runs in canonical order;
//  * batches of 32 candidates (lane p: candidate 32b + p): each lane's S row
//    arrives by ONE 1-D bulk copy (TMA engine; no LSU gather wavefronts) in a
//    double-buffered per-warp staging area while the previous batch runs its
//    canonical chains (dot_seq_dev's fmaf order) from shared memory; the row
//    pitch is an odd number of 16-byte units, so the lanes' 128-bit reads are
//    conflict-free;
//  * matches are written back IN PLACE, compacted, as (j << 32 | sim bits)
//    at the row's candidate offset (writes trail the reads), and
//    rowcount[i] = matches.
// Rows above kRowSortCap candidates are rechecked in grouped order (the big
// row sort orders them).  Requires dim % 4 == 0 and 16-byte aligned rows.
constexpr int kRowSortCap = 1024;

template <int E>
__device__ __forceinline__ void warp_sort_u32(uint32_t (&v)[E]) {
  const int lane = threadIdx.x & 31;
  constexpr int N = 32 * E;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j >= 1; j >>= 1) {
      if (j >= 32) {
        const int rj = j >> 5;
#pragma unroll
        for (int r = 0; r < E; r++) {
          if (r & rj) continue;
          const bool asc = ((32 * r + lane) & k) == 0;
          const uint32_t x = v[r], y = v[r | rj];
          const bool sw = asc ? (y < x) : (x < y);
          v[r] = sw ? y : x;
          v[r | rj] = sw ? x : y;
        }
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int r = 0; r < E; r++) {
          const bool asc = ((32 * r + lane) & k) == 0;
          const uint32_t y = __shfl_xor_sync(0xffffffffu, v[r], j);
          const uint32_t mnv = min(v[r], y), mxv = max(v[r], y);
          v[r] = (asc == lower) ? mnv : mxv;
        }
      }
    }
  }
}

// keys[c0 .. c0 + n) low halves sorted into list[0 .. n) (n <= 32 E)
template <int E>
__device__ __forceinline__ void sort_row_js(const uint64_t* __restrict__ keys, uint64_t c0, int n,
                                            uint32_t* list) {
  const int lane = threadIdx.x & 31;
  uint32_t v[E];
#pragma unroll
  for (int r = 0; r < E; r++) {
    const int t = 32 * r + lane;
    v[r] = t < n ? (uint32_t)keys[c0 + t] : ~0u;
  }
  warp_sort_u32<E>(v);
#pragma unroll
  for (int r = 0; r < E; r++) list[32 * r + lane] = v[r];
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Staging of one 32-candidate batch: 8 groups of 4 rows.  kG4: one
// tile::gather4 tensor copy per group (lane 0 issues 8 per batch instead of
// 32 per-lane 1-D copies, whose uniform-register operands make the compiler
// loop over the lanes); a tensor copy's destination must be 128-byte
// aligned, so groups are 128-byte padded (rows within a group at pitch dim).
// Otherwise: per-lane 1-D bulk copies at a pitch of an odd number of 16-byte
// units (conflict-free 128-bit reads).
__host__ __device__ inline int rows_pitch(int dim, bool g4) {
  return g4 ? dim : (((dim / 4) & 1) ? dim : dim + 4);
}
__host__ __device__ inline int rows_group_bytes(int dim, bool g4) {
  return g4 ? (int)round_up(16 * dim, 128) : 16 * rows_pitch(dim, false);
}
// dynamic shared memory per warp: 2 batch buffers, 2 mbarriers, the sorted
// list (+128 for aligning the staging area)
__host__ __device__ inline int rows_warp_smem(int dim, bool g4) {
  return 2 * 8 * rows_group_bytes(dim, g4) + 16 + kRowSortCap * 4;
}

__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int c, uint32_t r0,
                                            uint32_t r1, uint32_t r2, uint32_t r3, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

#if SJB_AB_KERNELS
template <bool kG4>
__global__ void __launch_bounds__(256, 1)
recheck_rows_kernel(uint64_t* __restrict__ keys, const uint64_t* __restrict__ rowoff,
                    int64_t n_rows, const float* __restrict__ l32, const float* __restrict__ r32,
                    int dim, float theta, uint32_t* __restrict__ rowcount,
                    unsigned int* __restrict__ work, const __grid_constant__ CUtensorMap rmap) {
  extern __shared__ __align__(16) uint8_t rsm[];
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gbytes = rows_group_bytes(dim, kG4), bufbytes = 8 * gbytes;
  const int pitch = rows_pitch(dim, kG4);
  // staging first (128-byte aligned), then mbarriers, then the lists
  uint8_t* base = rsm + ((128 - (smem_u32(rsm) & 127)) & 127);
  uint8_t* stage = base + (size_t)warp * 2 * bufbytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + (size_t)nw * 2 * bufbytes) + 2 * warp;
  uint32_t* list = reinterpret_cast<uint32_t*>(base + (size_t)nw * 2 * bufbytes + 16 * nw) +
                   warp * kRowSortCap;
  // lane p's row in buffer b: group p / 4, row p % 4
  uint8_t* myrow0 = stage + (lane >> 2) * gbytes + (lane & 3) * pitch * 4;
  auto myrow = [&](int buf) { return reinterpret_cast<float*>(myrow0 + buf * bufbytes); };
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  fence_mbar_init();
  __syncwarp();
  const uint64_t pol = policy_evict_last();   // S rows: re-read by the rows of their cluster
  const uint32_t rowbytes = (uint32_t)dim * 4;
  const int nq = dim >> 2;
  uint32_t phase = 0;
  for (;;) {
    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(work, 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if ((int64_t)i >= n_rows) break;
    const uint64_t c0 = rowoff[i], n = rowoff[i + 1] - c0;
    if (n == 0) {
      if (lane == 0) rowcount[i] = 0u;
      continue;
    }
    const bool small = n <= (uint64_t)kRowSortCap;
    if (small) {
      const int m = (int)n;
      if (m <= 32) sort_row_js<1>(keys, c0, m, list);
      else if (m <= 64) sort_row_js<2>(keys, c0, m, list);
      else if (m <= 128) sort_row_js<4>(keys, c0, m, list);
      else if (m <= 256) sort_row_js<8>(keys, c0, m, list);
      else if (m <= 512) sort_row_js<16>(keys, c0, m, list);
      else sort_row_js<32>(keys, c0, m, list);
      __syncwarp();
    }
    const float4* a4 = reinterpret_cast<const float4*>(l32 + (size_t)i * dim);
    const uint64_t nb = (n + 31) >> 5;
    // batch b -> buffer b & 1; returns this lane's right offset
    auto issue = [&](uint64_t b) -> uint32_t {
      const int buf = (int)(b & 1);
      const uint64_t k = b * 32 + lane;
      const uint32_t cnt = (uint32_t)mn<uint64_t>(32, n - b * 32);
      uint32_t j = 0;
      if (k < n) j = small ? list[k] : (uint32_t)keys[c0 + k];
      fence_proxy_async_smem();   // this buffer's previous reads precede the copy
      __syncwarp();
      if (kG4) {
        // pad the last group with its first row (copied, never read)
        const uint32_t jp = __shfl_sync(0xffffffffu, j, (int)((cnt - 1) & ~3u));
        if (k >= n) j = jp;
        const uint32_t groups = (cnt + 3) >> 2;
        if (lane == 0) mbar_arrive_expect_tx(bar + buf, groups * 4 * rowbytes);
#pragma unroll
        for (int g = 0; g < 8; g++) {
          const uint32_t j0 = __shfl_sync(0xffffffffu, j, 4 * g);
          const uint32_t j1 = __shfl_sync(0xffffffffu, j, 4 * g + 1);
          const uint32_t j2 = __shfl_sync(0xffffffffu, j, 4 * g + 2);
          const uint32_t j3 = __shfl_sync(0xffffffffu, j, 4 * g + 3);
          if (lane == 0 && (uint32_t)g < groups)
            tma_gather4(stage + buf * bufbytes + g * gbytes, &rmap, 0, j0, j1, j2, j3, bar + buf,
                        pol);
        }
      } else {
        if (lane == 0) mbar_arrive_expect_tx(bar + buf, cnt * rowbytes);
        __syncwarp();
        if (k < n)
          bulk_g2s(myrow(buf), r32 + (size_t)j * dim, rowbytes, bar + buf, pol);
      }
      return j;
    };
    uint32_t j_cur = issue(0);
    uint32_t kept = 0;
    for (uint64_t b = 0; b < nb; b++) {
      const uint32_t j_next = b + 1 < nb ? issue(b + 1) : 0u;
      const int buf = (int)(b & 1);
      mbar_wait(bar + buf, (phase >> buf) & 1u);
      phase ^= 1u << buf;
      const uint64_t k = b * 32 + lane;
      float x = 0.0f;
      if (k < n) {
        const float4* s4 = reinterpret_cast<const float4*>(myrow(buf));
#pragma unroll 5
        for (int q = 0; q < nq; q++) {
          const float4 s = s4[q], r = __ldg(a4 + q);
          x = __fmaf_rn(r.x, s.x, x);
          x = __fmaf_rn(r.y, s.y, x);
          x = __fmaf_rn(r.z, s.z, x);
          x = __fmaf_rn(r.w, s.w, x);
        }
      }
      const bool ok = k < n && x >= theta;
      const uint32_t bal = __ballot_sync(0xffffffffu, ok);
      if (ok) keys[c0 + kept + __popc(bal & lanemask_lt())] = (uint64_t(j_cur) << 32) | __float_as_uint(x);
      kept += __popc(bal);
      j_cur = j_next;
    }
    __syncwarp();
    if (lane == 0) rowcount[i] = kept;
  }
}

#endif  // SJB_AB_KERNELS

#if SJB_AB_KERNELS
// Each row's matches (sorted, compacted at its candidate offset coff[i]) to
// the MatchSet columns at its match offset moff[i]; rows that were too long
// to sort go to the big-row list with their keys at moff[i] of bigkeys.
__global__ void __launch_bounds__(256)
emit_rows_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ coff,
                 const uint64_t* __restrict__ moff, int64_t n_rows, uint64_t* __restrict__ lefts,
                 uint64_t* __restrict__ rights, float* __restrict__ sims,
                 uint64_t* __restrict__ bigkeys, uint32_t* __restrict__ big_rows,
                 unsigned int* __restrict__ n_big, uint64_t left_base) {
  if (n_big[1] == 0) return;  // gate: outputs would overflow
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t i = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); i < n_rows;
       i += (int64_t)gridDim.x * wpb) {
    const uint64_t m0 = moff[i], kept = moff[i + 1] - m0;
    if (kept == 0) continue;
    const uint64_t c0 = coff[i];
    if (coff[i + 1] - c0 > (uint64_t)kRowSortCap) {
      if (lane == 0) big_rows[atomicAdd(n_big, 1u)] = (uint32_t)i;
      for (uint64_t t = lane; t < kept; t += 32) bigkeys[m0 + t] = keys[c0 + t];
      continue;
    }
    const uint64_t ir = left_base + (uint64_t)i;
    for (uint64_t t = lane; t < kept; t += 32) {
      const uint64_t key = keys[c0 + t];
      lefts[m0 + t] = ir;
      rights[m0 + t] = key >> 32;
      sims[m0 + t] = __uint_as_float((uint32_t)key);
    }
  }
}

#endif  // SJB_AB_KERNELS

// ----------------------------------- dense recheck, cluster-blocked rows
// The staged per-candidate recheck above is bound by the bytes it can keep
// in flight from L2 (32 GB of S rows at cfg5 theta = 0.4, ~5 ms).  Dense
// joins of clustered data re-read the same S rows: the left rows of one
// cluster match (nearly) the same right rows.  So:
//  1. count_rows also takes each row's signature = its smallest right offset;
//  2. rows grouped by signature (counting sort over hashed buckets: bucket,
//     scan, scatter), so consecutive rows tend to share their candidates;
//  3. recheck_blocks: a CTA takes up to 32 consecutive rows of one bucket, builds
//     the UNION of their right offsets (shared-memory hash set), and -- when
//     the block is dense (candidates >= kBlkDense x rows x union) -- stages
//     each union S row ONCE (1-D bulk copies) and the 32 R rows, and runs the
//     canonical chains with lane = left row and the S row a shared-memory
//     broadcast: eight union rows per step (independent chains sharing the R
//     row's 128-bit reads), every read conflict-free.  Each similarity goes to
//     its candidate's slot of the sorted row, recorded per (union row, row)
//     in a per-CTA global scratch while the masks are built.  Sparse blocks
//     (or unions above kBlkUnion) run the per-candidate staged recheck
//     instead, one warp per row;
//     Every row of <= kRowSortCap candidates is first sorted by right offset
//     in registers and written back (the canonical order the slots follow);
//  4. emit_sims: per row, the rechecked slots compacted into the MatchSet.
template <bool kWarp, class T>
__device__ void smem_bitonic(T* s, int n, int tid, int nthr);

constexpr int kBlkRows = 32;
constexpr int kBlkThreads = 256;
constexpr int kBlkWarps = kBlkThreads / 32;
constexpr int kBlkHashBits = 12;
constexpr int kBlkHash = 1 << kBlkHashBits;   // holds <= kBlkUnion + kBlkThreads keys
constexpr int kBlkUnion = 1024;
constexpr float kBlkDense = 0.25f;
constexpr int kBlkChains = 8;       // union rows per step of a warp
constexpr uint32_t kHashEmpty = 0xFFFFFFFFu;
#ifndef SJB_BLK_STATS
#define SJB_BLK_STATS 0
#endif
#if SJB_BLK_STATS
// diagnostics (-DSJB_BLK_STATS=1): dense / big / union-overflow / low-density
// blocks, candidates in dense and sparse blocks, summed dense unions
__device__ unsigned long long g_blk_stats[16];   // [8..15]: cycles per phase (CTA thread 0)
#define BLK_MARK(k)                                                   \
  do {                                                                \
    if (tid == 0) {                                                   \
      const long long now_ = clock64();                               \
      atomicAdd(&g_blk_stats[8 + (k)], (unsigned long long)(now_ - t_mark)); \
      t_mark = now_;                                                  \
    }                                                                 \
  } while (0)
#else
#define BLK_MARK(k) do { } while (0)
#endif

// Rows are grouped, not sorted, by signature: bucket = a multiplicative hash
// of it over nbk - 1 buckets (the last one for big and empty rows).  Equal
// signatures share a bucket; distinct ones rarely do (k distinct signatures
// collide ~k^2 / 2 nbk times), whereas contiguous ranges of signatures would
// merge clusters whose smallest members are neighbours -- and the rows of a
// shared bucket interleave, so every block of two such clusters overflows.
__device__ __forceinline__ uint32_t sig_bucket(uint32_t s, int shift, int64_t nbk) {
  (void)shift;
  if (nbk < 2) return 0u;
  if (s == ~0u) return (uint32_t)(nbk - 1);
  const uint32_t h = (uint32_t)(((uint64_t)s * 0x9E3779B97F4A7C15ull) >> 32);
  return (uint32_t)(((uint64_t)h * (uint64_t)(nbk - 1)) >> 32);
}
// empty rows and rows above kRowSortCap candidates share the last bucket
__device__ __forceinline__ uint32_t row_sig(const uint32_t* sig, const uint32_t* ccnt,
                                            int64_t i) {
  const uint32_t n = ccnt[i];
  return (n == 0 || n > (uint32_t)kRowSortCap) ? ~0u : sig[i];
}
__global__ void sig_hist_kernel(const uint32_t* __restrict__ sig,
                                const uint32_t* __restrict__ ccnt, int64_t n, int shift,
                                uint32_t* __restrict__ hist) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(hist + sig_bucket(row_sig(sig, ccnt, i), shift, n), 1u);
}
__global__ void sig_scatter_kernel(const uint32_t* __restrict__ sig,
                                   const uint32_t* __restrict__ ccnt, int64_t n, int shift,
                                   unsigned long long* __restrict__ cursor,
                                   uint32_t* __restrict__ perm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    perm[atomicAdd(cursor + sig_bucket(row_sig(sig, ccnt, i), shift, n), 1ull)] = (uint32_t)i;
}

// Candidate offsets in the order of the blocks: pcnt[p] = ccnt[perm[p]]
// (scanned into poff), then each row's start: start[perm[p]] = poff[p].  The
// grouping then lays every block's candidates out contiguously.
__global__ void perm_counts_kernel(const uint32_t* __restrict__ perm,
                                   const uint32_t* __restrict__ ccnt, int64_t n,
                                   uint32_t* __restrict__ pcnt) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    pcnt[p] = ccnt[perm[p]];
}
__global__ void perm_starts_kernel(const uint32_t* __restrict__ perm,
                                   const uint64_t* __restrict__ poff, int64_t n,
                                   uint64_t* __restrict__ start) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    start[perm[p]] = poff[p];
}

// the u32 right offsets g[c0 .. c0 + n) sorted in place (registers)
template <int E>
__device__ __forceinline__ void sort_js_back(uint32_t* __restrict__ g, uint64_t c0, int n) {
  const int lane = threadIdx.x & 31;
  uint32_t v[E];
#pragma unroll
  for (int r = 0; r < E; r++) {
    const int t = 32 * r + lane;
    v[r] = t < n ? g[c0 + t] : ~0u;
  }
  warp_sort_u32<E>(v);
#pragma unroll
  for (int r = 0; r < E; r++) {
    const int t = 32 * r + lane;
    if (t < n) g[c0 + t] = v[r];
  }
}
__device__ __forceinline__ void sort_js_dispatch(uint32_t* g, uint64_t c0, int m) {
  if (m <= 32) sort_js_back<1>(g, c0, m);
  else if (m <= 64) sort_js_back<2>(g, c0, m);
  else if (m <= 128) sort_js_back<4>(g, c0, m);
  else if (m <= 256) sort_js_back<8>(g, c0, m);
  else if (m <= 512) sort_js_back<16>(g, c0, m);
  else sort_js_back<32>(g, c0, m);
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Blocks never span two buckets: bucket b (rows [end_b - cnt_b, end_b) of
// the order, `cursor` holding the ends after the scatter) becomes
// ceil(cnt_b / 32) blocks, appended in any order: desc = start | count << 32.
__global__ void sig_blocks_kernel(const uint32_t* __restrict__ hist,
                                  const uint64_t* __restrict__ ends, int64_t nbk,
                                  uint64_t* __restrict__ desc, unsigned int* __restrict__ n_desc) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbk;
       b += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t cnt = hist[b];
    if (cnt == 0) continue;
    const uint64_t start = ends[b] - cnt;
    const uint32_t nb = (cnt + kBlkRows - 1) / kBlkRows;
    const uint32_t base = atomicAdd(n_desc, nb);
    for (uint32_t k = 0; k < nb; k++)
      desc[base + k] = (start + (uint64_t)k * kBlkRows) |
                       ((uint64_t)mn<uint32_t>(kBlkRows, cnt - k * kBlkRows) << 32);
  }
}

// shared memory: staging area of kBlkStage rows (sparse: warps 0..4 x 32
// rows; dense: 32 R rows + a window of 148 union S rows), then the fixed
// part (41 KB): 113 KB at d = 100, two CTAs per SM
constexpr int kBlkStage = 180;
constexpr int kBlkSparseWarps = kBlkStage / 32;
static_assert(kBlkStage + kBlkRows <= kBlkThreads, "one copy-issuing thread per staged row");
// (at least 64 KB: the area is also the block's j cache, ~13k candidates at
// cfg5 -- small dims would otherwise send every block to the sparse path)
__host__ __device__ inline int blk_stage_bytes(int dim) {
  return mx(kBlkStage * rows_pitch(dim, false) * 4, 64 * 1024);
}
__host__ __device__ inline int blk_window_rows(int dim) { return kBlkStage - kBlkRows; }
// Sort a[0 .. U) (U <= kBlkUnion, u32, distinct keys; tmp: kBlkUnion
// words, clobbered) by kBlkThreads threads: each warp sorts a run of 128 in
// registers (bitonic, no barriers), then runs merge pairwise (128 -> 1024):
// an element's place = its index + its rank in the other run (lower bound
// from the left run, upper bound from the right: the ~0 padding ties stay
// stable).  Three barriers per round instead of the 55 stages of a shared
// bitonic network.  Leaves the result in a.
__device__ void block_sort_u32(uint32_t* a, uint32_t* tmp, int U) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Up = (U + 127) & ~127;
  if (warp * 128 < Up) {
    uint32_t v[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int k = warp * 128 + 32 * r + lane;
      v[r] = k < U ? a[k] : ~0u;
    }
    warp_sort_u32<4>(v);
#pragma unroll
    for (int r = 0; r < 4; r++) a[warp * 128 + 32 * r + lane] = v[r];
  }
  __syncthreads();
  uint32_t* src = a;
  uint32_t* dst = tmp;
  for (int L = 128; L < Up; L <<= 1) {
    for (int k = tid; k < Up; k += kBlkThreads) {
      const int base = k & ~(2 * L - 1), off = k - base;
      const bool left = off < L;
      const uint32_t x = src[k];
      // rank of x in the other run (bounded by the elements that exist)
      const int ob = left ? base + L : base;
      const int on = left ? min(L, Up - (base + L)) : L;
      int lo = 0, hi = max(on, 0);
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const uint32_t y = src[ob + mid];
        if (left ? (y < x) : (y <= x)) lo = mid + 1; else hi = mid;
      }
      dst[base + (left ? off : off - L) + lo] = x;
    }
    __syncthreads();
    uint32_t* t = src;
    src = dst;
    dst = t;
  }
  if (src != a) {
    for (int k = tid; k < U; k += kBlkThreads) a[k] = src[k];
    __syncthreads();
  }
}

struct BlkShared {
  uint32_t hkeys[kBlkHash];
  uint32_t hmask[kBlkHash];   // per hash slot: bit r <=> row r has the key
  uint32_t uniq[kBlkUnion];
  uint32_t mask[kBlkUnion];
  uint64_t c0[kBlkRows];
  uint32_t n[kBlkRows], off[kBlkRows], row[kBlkRows], kept[kBlkRows], rank[2][kBlkRows];
  uint64_t sbar[kBlkWarps];
  uint64_t dbar;
  uint32_t item, next, count, ucnt, ovf, big, cand;
};
__host__ __device__ inline int blk_smem_bytes(int dim) {
  return blk_stage_bytes(dim) + (int)sizeof(BlkShared) + 16;
}

__global__ void __launch_bounds__(kBlkThreads)
recheck_blocks_kernel(uint32_t* __restrict__ g32, const uint64_t* __restrict__ poff,
                      const uint32_t* __restrict__ ccnt, uint64_t* __restrict__ keys,
                      const uint32_t* __restrict__ perm, const uint64_t* __restrict__ desc,
                      const unsigned int* __restrict__ n_desc,
                      const float* __restrict__ l32, const float* __restrict__ r32, int dim,
                      float theta, uint32_t* __restrict__ rowcount,
                      unsigned int* __restrict__ work) {
  extern __shared__ __align__(16) uint8_t bsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pitch = rows_pitch(dim, false), nq = dim >> 2;
  const uint32_t rowbytes = (uint32_t)dim * 4;
  float* stage = reinterpret_cast<float*>(bsm);
  BlkShared& sh = *reinterpret_cast<BlkShared*>(bsm + blk_stage_bytes(dim));
  const int win = blk_window_rows(dim);
  const uint32_t jcap = (uint32_t)blk_stage_bytes(dim) / 4;   // j cache entries
  uint32_t* jc = reinterpret_cast<uint32_t*>(bsm);
  if (tid < kBlkWarps) mbar_init(&sh.sbar[tid], 1);
  if (tid == 0) mbar_init(&sh.dbar, 1);
  fence_mbar_init();
  __syncthreads();
  const uint64_t pol = policy_evict_last();
  uint32_t sphase = 0, dphase = 0;
#if SJB_BLK_STATS
  long long t_mark = clock64();
#endif
  const unsigned int nd = *n_desc;
  if (tid == 0) sh.next = atomicAdd(work, 1u);
  for (;;) {
    if (tid == 0) {
      sh.item = sh.next;
      sh.next = atomicAdd(work, 1u);
    }
    if (tid < kBlkRows) sh.kept[tid] = 0u;
    __syncthreads();
    BLK_MARK(0);
    if (sh.item >= nd) break;
    const uint64_t dsc = desc[sh.item];
    const int64_t p0 = (int64_t)(uint32_t)dsc;
    const int nrows = (int)(dsc >> 32);
    if (tid == 32 && sh.next < nd) {
      // the next block's candidates (contiguous in the blocks' order) on
      // their way to L2 while this block runs
      const uint64_t dn = desc[sh.next];
      const int64_t q0 = (int64_t)(uint32_t)dn;
      const uint64_t a = poff[q0] & ~3ull, b = (poff[q0 + (int64_t)(dn >> 32)] + 3) & ~3ull;
      for (uint64_t x = a; x < b; x += 8192)
        prefetch_l2_bulk(g32 + x, (uint32_t)mn<uint64_t>(32768, (b - x) * 4));
    }
    if (tid < kBlkRows) {
      uint32_t i = 0, n = 0;
      uint64_t c0 = 0;
      if (tid < nrows) {
        i = perm[p0 + tid];
        c0 = poff[p0 + tid];
        n = ccnt[i];
      }
      sh.row[tid] = i;
      sh.c0[tid] = c0;
      sh.n[tid] = n;
      // block totals and the rows' offsets in the shared j cache (warp 0)
      const uint32_t nc = mn<uint32_t>(n, 1u << 20);
      uint32_t incl = nc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += y;
      }
      sh.off[tid] = incl - nc;
      const uint32_t cand = __shfl_sync(0xffffffffu, incl, 31);
      const bool big = __any_sync(0xffffffffu, n > (uint32_t)kRowSortCap);
      if (tid == 0) {
        sh.cand = cand;
        sh.big = big ? 1u : 0u;
        sh.count = 0u;
        // the block's right offsets (+ 16-byte alignment slack) must fit
        // the j cache (the staging area)
        sh.ovf = (big || cand == 0 || cand + 8 > jcap) ? 1u : 0u;
      }
    }
    for (int h = tid; h < kBlkHash; h += kBlkThreads) {
      sh.hkeys[h] = kHashEmpty;
      sh.hmask[h] = 0u;
    }
    __syncthreads();
    BLK_MARK(1);
    // ---- union of the block's right offsets: a shared-memory hash set
    // (gives up above kBlkUnion keys).  The block's j's are cached in the
    // staging area on the way (row r at off[r]); each lane loads four
    // before inserting them, and looks before it CASes (the rows of a block
    // mostly share their keys).
    auto hash_of = [](uint32_t j) { return (j * 0x9E3779B1u) >> (32 - kBlkHashBits); };
    const uint32_t jhead = (uint32_t)(sh.c0[0] & 3u);
    const uint32_t* jcb = jc + jhead;
    if (!sh.ovf) {
      // (a) the j cache: the block's candidates are contiguous (grouped in
      // the blocks' order) -- one bulk copy of the 16-byte aligned span;
      // candidate k of the block is jcb[k]
      if (tid == 0) {
        const uint32_t bytes = ((jhead + sh.cand + 3) & ~3u) * 4;
        mbar_arrive_expect_tx(&sh.dbar, bytes);
        bulk_g2s(jc, g32 + (sh.c0[0] - jhead), bytes, &sh.dbar, pol);
      }
      mbar_wait(&sh.dbar, dphase);
      dphase ^= 1u;
      // (b) insert in cache order: the CTA's threads walk ~one row at a time,
      // so concurrent inserts are distinct keys, and the later rows mostly
      // find theirs (a read, no CAS)
      // and each candidate's row bit set in its key's slot (the membership
      // masks, indexed by slot until the union is sorted)
      const uint32_t C = sh.cand;
      int r = 0;
      for (uint32_t k = tid; k < C; k += kBlkThreads) {
        if (*(volatile uint32_t*)&sh.ovf) break;
        while (r + 1 < nrows && k >= sh.off[r + 1]) r++;
        const uint32_t j = jcb[k];
        uint32_t h = hash_of(j);
        for (;;) {
          uint32_t cur = sh.hkeys[h];
          if (cur == kHashEmpty) {
            cur = atomicCAS(&sh.hkeys[h], kHashEmpty, j);
            if (cur == kHashEmpty) {
              if (atomicAdd(&sh.count, 1u) >= (uint32_t)kBlkUnion) sh.ovf = 1u;
              break;
            }
          }
          if (cur == j) break;
          h = (h + 1) & (kBlkHash - 1);
        }
        atomicOr(&sh.hmask[h], 1u << r);
      }
    }
    __syncthreads();
    BLK_MARK(2);
    const uint32_t U = sh.count;
    const bool dense = !sh.ovf && U > 0 && (float)sh.cand >= kBlkDense * (float)nrows * (float)U;
#if SJB_BLK_STATS
    if (tid == 0) {
      atomicAdd(&g_blk_stats[dense ? 0 : (sh.big ? 1 : (sh.ovf ? 2 : 3))], 1ull);
      atomicAdd(&g_blk_stats[dense ? 4 : 5], (unsigned long long)sh.cand);
      if (dense) atomicAdd(&g_blk_stats[6], (unsigned long long)U);
    }
#endif
    if (dense) {
      // the union sorted (ascending right offsets), each key's sorted index
      // recorded in its hash slot
      if (tid == 0) sh.ucnt = 0u;
      __syncthreads();
      for (int h = tid; h < kBlkHash; h += kBlkThreads) {
        const uint32_t k = sh.hkeys[h];
        if (k != kHashEmpty) sh.uniq[atomicAdd(&sh.ucnt, 1u)] = k;
      }
      __syncthreads();
      block_sort_u32(sh.uniq, sh.mask, (int)U);   // (mask: scratch, written next)
      // membership in sorted order: bit r of mask[u] <=> (row r, uniq[u]) is
      // a candidate
      for (uint32_t u = tid; u < U; u += kBlkThreads) {
        const uint32_t j = sh.uniq[u];
        uint32_t h = hash_of(j);
        while (sh.hkeys[h] != j) h = (h + 1) & (kBlkHash - 1);
        sh.mask[u] = sh.hmask[h];
      }
      if (tid < kBlkRows) sh.rank[0][tid] = 0u;
      __syncthreads();
      BLK_MARK(3);
      const float* Rs = stage;
      const float* Ss = stage + (size_t)kBlkRows * pitch;
      const float4* R4 = reinterpret_cast<const float4*>(Rs + (size_t)lane * pitch);
      const uint64_t c0 = sh.c0[lane];
      uint32_t kept = 0;
      int wpar = 0;
      for (uint32_t u0 = 0; u0 < U; u0 += (uint32_t)win) {
        const uint32_t u1 = mn<uint32_t>(U, u0 + (uint32_t)win);
        fence_proxy_async_smem();
        __syncthreads();   // masks complete (and the j cache dead) / the previous window consumed
        BLK_MARK(u0 == 0 ? 4 : 6);
        if (tid == 0)
          mbar_arrive_expect_tx(&sh.dbar, (u1 - u0) * rowbytes + (u0 == 0 ? nrows * rowbytes : 0u));
        __syncthreads();
        if (tid < (int)(u1 - u0))
          bulk_g2s(stage + (size_t)(kBlkRows + tid) * pitch,
                   r32 + (size_t)sh.uniq[u0 + tid] * dim, rowbytes, &sh.dbar, pol);
        if (u0 == 0 && tid >= kBlkStage && tid - kBlkStage < nrows) {
          const int r = tid - kBlkStage;
          bulk_g2s(stage + (size_t)r * pitch, l32 + (size_t)sh.row[r] * dim, rowbytes, &sh.dbar,
                   pol);
        }
        mbar_wait(&sh.dbar, dphase);
        dphase ^= 1u;
        BLK_MARK(5);
        // warp w: a contiguous run of the window's groups of kBlkChains union
        // rows; lane = row.  The union is sorted, so row r's candidate at
        // union row u is its rank-th: rank = bit r set in the masks before u
        // (a running count); the chains of a group are independent and
        // share the R row's reads.  Result: keys[c0 + rank] = j << 32 | sim.
        const uint32_t groups = (u1 - u0 + kBlkChains - 1) / kBlkChains;
        const uint32_t ua = mn<uint32_t>(u1, u0 + kBlkChains * (groups * warp / kBlkWarps));
        const uint32_t ub = mn<uint32_t>(u1, u0 + kBlkChains * (groups * (warp + 1) / kBlkWarps));
        uint32_t rank = sh.rank[wpar][lane];
        for (uint32_t u = u0; u < ua; u++) rank += (sh.mask[u] >> lane) & 1u;
        const int p4 = pitch >> 2;
        for (uint32_t u = ua; u < ub; u += kBlkChains) {
          uint32_t m[kBlkChains], any = 0u;
#pragma unroll
          for (int c = 0; c < kBlkChains; c++) {
            m[c] = u + c < ub ? sh.mask[u + c] : 0u;
            any |= m[c];
          }
          if (any == 0u) continue;
          // union rows u .. u + kBlkChains - 1 at a constant pitch (rows past
          // ub read staged or scratch words; their results are dropped)
          const float4* S4 = reinterpret_cast<const float4*>(Ss + (size_t)(u - u0) * pitch);
          float x[kBlkChains];
#pragma unroll
          for (int c = 0; c < kBlkChains; c++) x[c] = 0.0f;
#pragma unroll 5
          for (int q = 0; q < nq; q++) {
            const float4 a = R4[q];
#pragma unroll
            for (int c = 0; c < kBlkChains; c++) {
              const float4 b = S4[c * p4 + q];
              x[c] = __fmaf_rn(a.x, b.x, x[c]);
              x[c] = __fmaf_rn(a.y, b.y, x[c]);
              x[c] = __fmaf_rn(a.z, b.z, x[c]);
              x[c] = __fmaf_rn(a.w, b.w, x[c]);
            }
          }
#pragma unroll
          for (int c = 0; c < kBlkChains; c++) {
            if ((m[c] >> lane) & 1u) {
              const bool ok = x[c] >= theta;
              keys[c0 + rank] = ((uint64_t)sh.uniq[u + c] << 32) |
                                (ok ? __float_as_uint(x[c]) : kRejected);
              rank++;
              kept += ok ? 1u : 0u;
            }
          }
        }
        // the rank at the window's end, for the next window (the other
        // parity: this window's readers may still be reading theirs)
        if (warp == kBlkWarps - 1) sh.rank[wpar ^ 1][lane] = rank;
        wpar ^= 1;
      }
      if (kept) atomicAdd(&sh.kept[lane], kept);
    } else {
      // ---- sparse block: per-candidate staged recheck, one warp per row
      float* buf = stage + (size_t)warp * 32 * pitch;
      float* myrow = buf + (size_t)lane * pitch;
      for (int r = warp; r < nrows && warp < kBlkSparseWarps; r += kBlkSparseWarps) {
        const uint64_t c0 = sh.c0[r];
        const uint32_t n = sh.n[r];
        if (n > 0 && n <= (uint32_t)kRowSortCap) {
          sort_js_dispatch(g32, c0, (int)n);
          __syncwarp();   // (the batches below read the sorted offsets back)
        }
        const float4* a4 = reinterpret_cast<const float4*>(l32 + (size_t)sh.row[r] * dim);
        uint32_t kept = 0;
        for (uint32_t b0 = 0; b0 < n; b0 += 32) {
          const uint32_t k = b0 + lane, cnt = mn<uint32_t>(32u, n - b0);
          const uint32_t j = k < n ? g32[c0 + k] : 0u;
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive_expect_tx(&sh.sbar[warp], cnt * rowbytes);
          __syncwarp();
          if (k < n) bulk_g2s(myrow, r32 + (size_t)j * dim, rowbytes, &sh.sbar[warp], pol);
          mbar_wait(&sh.sbar[warp], sphase);
          sphase ^= 1u;
          if (k < n) {
            const float4* s4 = reinterpret_cast<const float4*>(myrow);
            float x = 0.0f;
#pragma unroll 5
            for (int q = 0; q < nq; q++) {
              const float4 s = s4[q], a = __ldg(a4 + q);
              x = __fmaf_rn(a.x, s.x, x);
              x = __fmaf_rn(a.y, s.y, x);
              x = __fmaf_rn(a.z, s.z, x);
              x = __fmaf_rn(a.w, s.w, x);
            }
            const bool ok = x >= theta;
            keys[c0 + k] = ((uint64_t)j << 32) | (ok ? __float_as_uint(x) : kRejected);
            kept += ok ? 1u : 0u;
          }
        }
        kept = __reduce_add_sync(0xffffffffu, kept);
        if (lane == 0) sh.kept[r] = kept;
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    BLK_MARK(dense ? 6 : 7);
    if (tid < nrows) rowcount[sh.row[tid]] = sh.kept[tid];
  }
}

// Rechecked candidate slots (j << 32 | sim bits or kRejected; rows sorted;
// row i's at [cend[i] - ccnt[i], cend[i])) compacted into the MatchSet
// columns at the match offsets moff; big rows (unsorted) go to the big-row
// list with their keys at moff of bigkeys.
__global__ void __launch_bounds__(256)
emit_sims_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ cend,
                 const uint32_t* __restrict__ ccnt, const uint64_t* __restrict__ moff,
                 int64_t n_rows, uint64_t* __restrict__ lefts, uint64_t* __restrict__ rights,
                 float* __restrict__ sims, uint64_t* __restrict__ bigkeys,
                 uint32_t* __restrict__ big_rows, unsigned int* __restrict__ n_big,
                 uint64_t left_base) {
  if (n_big[1] == 0) return;  // gate: outputs would overflow
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t i = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); i < n_rows;
       i += (int64_t)gridDim.x * wpb) {
    const uint64_t m0 = moff[i];
    if (moff[i + 1] == m0) continue;
    const uint64_t n = ccnt[i], c0 = cend[i] - n;   // rows laid out in the blocks' order
    const bool big = n > (uint64_t)kRowSortCap;
    if (big && lane == 0) big_rows[atomicAdd(n_big, 1u)] = (uint32_t)i;
    const uint64_t ir = left_base + (uint64_t)i;
    uint64_t run = m0;
    // eight 32-candidate chunks per step: their loads in flight together
    for (uint64_t t0 = 0; t0 < n; t0 += 256) {
      uint64_t kv[8];
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const uint64_t t = t0 + 32 * e + lane;
        kv[e] = t < n ? keys[c0 + t] : (uint64_t)kRejected;
      }
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const uint32_t sb = (uint32_t)kv[e];
        const bool ok = sb != kRejected;
        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
        if (ok) {
          const uint64_t pos = run + __popc(bal & lt);
          if (big) {
            bigkeys[pos] = kv[e];
          } else {
            lefts[pos] = ir;
            rights[pos] = kv[e] >> 32;
            sims[pos] = __uint_as_float(sb);
          }
        }
        run += __popc(bal);
      }
    }
  }
}

// Matches of the grouped candidates into per-row runs (j << 32 | sim bits)
// at the match offsets (cursor = row offsets), for the segmented sort.
__global__ void compact_rows_kernel(const uint64_t* __restrict__ grouped,
                                    const uint32_t* __restrict__ sims_bits,
                                    const uint64_t* __restrict__ total,
                                    unsigned long long* __restrict__ cursor,
                                    uint64_t* __restrict__ keys,
                                    const unsigned int* __restrict__ gate) {
  if (gate[1] == 0) return;
  const uint64_t n = *total;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t sb = sims_bits[k];
    if (sb == kRejected) continue;
    const uint64_t u = grouped[k];
    keys[atomicAdd(cursor + (uint32_t)(u >> 32), 1ull)] = (uint64_t((uint32_t)u) << 32) | sb;
  }
}

__global__ void scatter_kernel(const uint64_t* __restrict__ cand, uint64_t seg_cap,
                               const unsigned long long* __restrict__ cta_count, int n_cta,
                               const uint32_t* __restrict__ sims_bits,
                               unsigned long long* __restrict__ cursor,
                               uint64_t* __restrict__ keys, const unsigned int* __restrict__ gate) {
  if (gate[1] == 0) return;
  const uint64_t total = (uint64_t)n_cta * seg_cap;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < total;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = p / seg_cap, local = p - c * seg_cap;
    const uint64_t cnt = mn<uint64_t>(cta_count[c], seg_cap);
    if (local >= cnt) continue;
    const uint32_t sb = sims_bits[p];
    if (sb == kRejected) continue;
    const uint64_t u = cand[p];
    const uint32_t i = (uint32_t)(u >> 32), j = (uint32_t)u;
    const uint64_t q = atomicAdd(cursor + i, 1ull);
    keys[q] = (uint64_t(j) << 32) | sb;
  }
}

// ------------------------------------------------------ segmented sort
// Bitonic network in its "mirror" form: every compare-exchange puts the
// smaller key at the lower index, so a segment of any length sorts with
// virtual +inf padding that never moves.
template <class T>
__device__ __forceinline__ void cmpx(T* s, int a, int b) {
  T x = s[a], y = s[b];
  if (y < x) {
    s[a] = y;
    s[b] = x;
  }
}

// Sort s[0..n) in shared memory with `nthr` cooperating threads (tid in
// [0, nthr)); `sync` is the barrier among them.
template <bool kWarp>
__device__ __forceinline__ void nsync() {
  if (kWarp) __syncwarp(); else __syncthreads();
}

// k and j are powers of two: block/offset by shift and mask (a runtime
// integer division per compare-exchange dominated the sort).
template <bool kWarp, class T>
__device__ void smem_bitonic(T* s, int n, int tid, int nthr) {
  int P = 1, lp = 0;
  while (P < n) {
    P <<= 1;
    lp++;
  }
  for (int lk = 1; lk <= lp; lk++) {
    const int k = 1 << lk, lh = lk - 1;  // k/2 = 1 << lh
    // mirror step
    for (int t = tid; t < P / 2; t += nthr) {
      const int blk = t >> lh, off = t & ((1 << lh) - 1);
      const int a = (blk << lk) + off, b = (blk << lk) + k - 1 - off;
      if (b < n) cmpx(s, a, b);
    }
    nsync<kWarp>();
    for (int lj = lk - 2; lj >= 0; lj--) {
      const int j = 1 << lj;
      for (int t = tid; t < P / 2; t += nthr) {
        const int blk = t >> lj, off = t & (j - 1);
        const int a = (blk << (lj + 1)) + off, b = a + j;
        if (b < n) cmpx(s, a, b);
      }
      nsync<kWarp>();
    }
  }
}

__device__ __forceinline__ void write_row(uint64_t i, const uint64_t* sorted, uint64_t q0, int n,
                                          int tid, int nthr, uint64_t* __restrict__ lefts,
                                          uint64_t* __restrict__ rights,
                                          float* __restrict__ sims) {
  for (int t = tid; t < n; t += nthr) {
    const uint64_t key = sorted[t];
    lefts[q0 + t] = i;
    rights[q0 + t] = key >> 32;
    sims[q0 + t] = __uint_as_float((uint32_t)key);
  }
}

constexpr int kSortWarpCap = 1024;  // rows up to this many keys: one warp
constexpr int kSortSmallThreads = 128;

// Bitonic sort of one row of n <= 32 E keys in a warp's registers: key
// i = 32 r + l lives in register r of lane l (coalesced loads and stores),
// padded with ~0, which no key equals (right offsets are < 2^32 and the sim
// bits of a match are never all-ones).  Steps with j < 32 compare-exchange
// across lanes (__shfl_xor), steps with j >= 32 inside a lane.  No
// shared-memory traffic.
template <int E>
__device__ __forceinline__ void warp_sort_row(const uint64_t* __restrict__ keys, uint64_t q0, int n,
                                              uint64_t i_row, uint64_t* __restrict__ lefts,
                                              uint64_t* __restrict__ rights,
                                              float* __restrict__ sims) {
  const int lane = threadIdx.x & 31;
  uint64_t v[E];
#pragma unroll
  for (int r = 0; r < E; r++) {
    const int i = 32 * r + lane;
    v[r] = i < n ? keys[q0 + i] : ~0ull;
  }
  constexpr int N = 32 * E;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j >= 1; j >>= 1) {
      if (j >= 32) {
        const int rj = j >> 5;
#pragma unroll
        for (int r = 0; r < E; r++) {
          if (r & rj) continue;
          const bool asc = ((32 * r + lane) & k) == 0;
          const uint64_t x = v[r], y = v[r | rj];
          const bool sw = asc ? (y < x) : (x < y);
          v[r] = sw ? y : x;
          v[r | rj] = sw ? x : y;
        }
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int r = 0; r < E; r++) {
          const bool asc = ((32 * r + lane) & k) == 0;
          const uint64_t y = __shfl_xor_sync(0xffffffffu, v[r], j);
          const uint64_t mnv = v[r] < y ? v[r] : y, mxv = v[r] < y ? y : v[r];
          v[r] = (asc == lower) ? mnv : mxv;
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < E; r++) {
    const int i = 32 * r + lane;
    if (i < n) {
      lefts[q0 + i] = i_row;
      rights[q0 + i] = v[r] >> 32;
      sims[q0 + i] = __uint_as_float((uint32_t)v[r]);
    }
  }
}

__global__ void __launch_bounds__(kSortSmallThreads)
segsort_small_kernel(const uint64_t* __restrict__ rowoff, int64_t n_rows, const uint64_t* __restrict__ keys,
                     uint64_t* __restrict__ lefts, uint64_t* __restrict__ rights,
                     float* __restrict__ sims, uint32_t* __restrict__ big_rows,
                     unsigned int* __restrict__ n_big, uint64_t left_base) {
  __shared__ uint64_t buf[kSortSmallThreads / 32][kSortWarpCap];
  if (n_big[1] == 0) return;  // gate: outputs would overflow
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wpb = kSortSmallThreads / 32;
  for (int64_t i = (int64_t)blockIdx.x * wpb + warp; i < n_rows; i += (int64_t)gridDim.x * wpb) {
    const uint64_t q0 = rowoff[i], q1 = rowoff[i + 1];
    const int64_t n = (int64_t)(q1 - q0);
    if (n == 0) continue;
    if (n > kSortWarpCap) {
      if (lane == 0) big_rows[atomicAdd(n_big, 1u)] = (uint32_t)i;
      continue;
    }
    const uint64_t ir = left_base + (uint64_t)i;
    const int m = (int)n;
    if (m <= 32) warp_sort_row<1>(keys, q0, m, ir, lefts, rights, sims);
    else if (m <= 64) warp_sort_row<2>(keys, q0, m, ir, lefts, rights, sims);
    else if (m <= 128) warp_sort_row<4>(keys, q0, m, ir, lefts, rights, sims);
    else if (m <= 256) warp_sort_row<8>(keys, q0, m, ir, lefts, rights, sims);
    else {
      // 257..1024 keys: the shared-memory network (measured faster there than
      // 16-32 registers per lane: cfg5 rows of ~400, 2.2 vs 2.5 ms)
      uint64_t* sm = buf[warp];
      for (int t = lane; t < m; t += 32) sm[t] = keys[q0 + t];
      __syncwarp();
      smem_bitonic<true>(sm, m, lane, 32);
      write_row(ir, sm, q0, m, lane, 32, lefts, rights, sims);
      __syncwarp();
    }
  }
}

constexpr int kSortBigThreads = 512;
constexpr int kSortBigCap = 26624;   // keys sorted whole in shared memory (208 KB)


// Rows longer than kSortWarpCap: one CTA per row.  Up to kSortBigCap keys
// sort whole in shared memory (bitonic).  Longer rows -- Zipf clusters give
// cfg4 rows with tens of thousands of matches -- are ranked instead of sorted:
// a row's right offsets j are distinct, so j's position in the row is the
// number of the row's keys below it.  Per window of kRankWindow offsets: set
// bit j of a shared-memory bitmap, prefix-popcount it per 1024-bit group and
// per word within the group (u16), and write each key straight to
// q0 + (keys in earlier windows) + rank: three shared reads per key.
constexpr int kRankWindow = 1 << 20;                  // bits: 128 KB of shared memory
constexpr int kRankWords = kRankWindow / 32;
constexpr int kRankSub = 8;                            // words per prefix group (256 bits)
constexpr int kRankGroups = kRankWords / kRankSub;     // 4096 groups
constexpr int kRankPer = kRankGroups / kSortBigThreads;   // consecutive groups scanned per thread
static_assert(kRankGroups % kSortBigThreads == 0 && kRankPer == 8, "group scan layout");
constexpr int kRankMetaBytes = (((kRankGroups + 1) * 4 + 64) + 15) / 16 * 16;   // gpre + warp sums
static_assert(kRankWords * 4 + kRankMetaBytes <= kSortBigCap * 8, "bitmap + prefixes fit the buffer");
// (Staging a window's placed keys in the rest of the buffer so the output
// columns are written in order was measured: no gain, 1.63 -> 1.7 ms at the
// cfg4 slice -- the scattered 20-byte writes are not what the kernel waits on.)

// Per window: clear the bitmap (16-byte stores), set the keys' bits, count each
// 8-word group (two 16-byte loads per group), exclusive-scan the 4096 group
// counts (8 consecutive counts per thread + one block scan), then place each
// key: group prefix + the popcounts of the <= 7 words before its word + the
// masked popcount of its word.  (A u16 prefix per WORD cost a pass over all
// 32768 words per window -- 25k warp instructions even with conflict-free
// warp-per-group scans -- for 3 reads per key; rows of a few thousand keys are
// far cheaper with 4096 prefixes and ~6 reads per key.)
// Keys are read in batches of kRankBatch independent loads per thread (one
// memory round trip per batch: ncu put 52% of this kernel's stall samples on
// the two loops' one-key-at-a-time loads); a row of <= kRankBatch * threads
// keys (4096) is loaded ONCE into registers and reused by both loops of every
// window (kSmall).
constexpr int kRankBatch = 8;
constexpr uint64_t kNoKey = ~0ull;   // right offset 2^32 - 1: outside every window

template <bool kSmall>
__device__ void rank_row(const uint64_t* __restrict__ g, int64_t n, uint64_t q0, uint64_t i_row,
                         int64_t n_right, uint32_t* bits, uint32_t* gpre,
                         uint64_t* __restrict__ lefts, uint64_t* __restrict__ rights,
                         float* __restrict__ sims) {
  uint32_t* wsum = gpre + kRankGroups + 1;   // per-warp totals of the block scan (16)
  const int tid = threadIdx.x, nthr = blockDim.x;   // nthr == kSortBigThreads
  const int lane = tid & 31, warp = tid >> 5;
  uint4* b4 = reinterpret_cast<uint4*>(bits);
  uint64_t base = 0;
  uint64_t kreg[kRankBatch];
  auto load_batch = [&](int64_t t0) {
#pragma unroll
    for (int u = 0; u < kRankBatch; u++) {
      const int64_t t = t0 + (int64_t)u * nthr;
      kreg[u] = t < n ? g[t] : kNoKey;
    }
  };
  if (kSmall) load_batch(tid);
  for (int64_t w0 = 0; w0 < n_right; w0 += kRankWindow) {
    for (int t = tid; t < kRankWords / 4; t += nthr) b4[t] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    for (int64_t t0 = tid; t0 < n; t0 += (int64_t)kRankBatch * nthr) {
      if (!kSmall) load_batch(t0);
#pragma unroll
      for (int u = 0; u < kRankBatch; u++) {
        const uint64_t o = (kreg[u] >> 32) - (uint64_t)w0;
        if (o < (uint64_t)kRankWindow) atomicOr(&bits[o >> 5], 1u << (o & 31));
      }
    }
    __syncthreads();
    // group counts: thread t counts groups t, t + nthr, ... (neighbouring
    // lanes read neighbouring 32-byte groups)
    for (int q = tid; q < kRankGroups; q += nthr) {
      const uint4 x = b4[2 * q], y = b4[2 * q + 1];
      gpre[q] = __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w) + __popc(y.x) +
                __popc(y.y) + __popc(y.z) + __popc(y.w);
    }
    __syncthreads();
    // exclusive scan: thread t owns counts 8t .. 8t + 7
    uint32_t c[kRankPer];
    {
      const uint4 x = reinterpret_cast<const uint4*>(gpre)[2 * tid];
      const uint4 y = reinterpret_cast<const uint4*>(gpre)[2 * tid + 1];
      c[0] = x.x; c[1] = x.y; c[2] = x.z; c[3] = x.w;
      c[4] = y.x; c[5] = y.y; c[6] = y.z; c[7] = y.w;
    }
    uint32_t tot = 0;
#pragma unroll
    for (int k = 0; k < kRankPer; k++) {
      const uint32_t v = c[k];
      c[k] = tot;
      tot += v;
    }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint32_t wbase = 0, all = 0;
    for (int w = 0; w < (nthr >> 5); w++) {
      const uint32_t v = wsum[w];
      if (w < warp) wbase += v;
      all += v;
    }
    const uint32_t tb = wbase + incl - tot;
    reinterpret_cast<uint4*>(gpre)[2 * tid] =
        make_uint4(tb + c[0], tb + c[1], tb + c[2], tb + c[3]);
    reinterpret_cast<uint4*>(gpre)[2 * tid + 1] =
        make_uint4(tb + c[4], tb + c[5], tb + c[6], tb + c[7]);
    __syncthreads();
    for (int64_t t0 = tid; t0 < n; t0 += (int64_t)kRankBatch * nthr) {
      if (!kSmall) load_batch(t0);
#pragma unroll
      for (int u = 0; u < kRankBatch; u++) {
        const uint64_t key = kreg[u];
        const uint64_t o = (key >> 32) - (uint64_t)w0;
        if (o >= (uint64_t)kRankWindow) continue;
        const uint32_t word = (uint32_t)(o >> 5), grp = word / kRankSub;
        uint32_t rank = gpre[grp] + __popc(bits[word] & ((1u << (o & 31)) - 1u));
        for (uint32_t w = grp * kRankSub; w < word; w++) rank += __popc(bits[w]);
        const uint64_t pos = q0 + base + rank;
        lefts[pos] = i_row;
        rights[pos] = key >> 32;
        sims[pos] = __uint_as_float((uint32_t)key);
      }
    }
    base += all;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSortBigThreads)
segsort_big_kernel(const uint64_t* __restrict__ rowoff, uint64_t* __restrict__ keys,
                   uint64_t* __restrict__ lefts, uint64_t* __restrict__ rights,
                   float* __restrict__ sims, const uint32_t* __restrict__ big_rows,
                   const unsigned int* __restrict__ n_big, uint64_t left_base, int64_t n_right) {
  extern __shared__ __align__(16) uint64_t sbuf[];
  if (n_big[1] == 0) return;  // gate: outputs would overflow
  const unsigned nb = n_big[0];
  // rows handed out by a counter (n_big[2], zero since join_begin): Zipf clusters
  // make a few rows ten times longer than the rest, and a static row -> CTA
  // map leaves the CTAs that drew them running alone at the end
  __shared__ unsigned s_row;
  unsigned int* next = const_cast<unsigned int*>(n_big) + 2;
  for (;;) {
    if (threadIdx.x == 0) s_row = atomicAdd(next, 1u);
    __syncthreads();
    const unsigned r = s_row;
    __syncthreads();
    if (r >= nb) break;
    const uint32_t i = big_rows[r];
    const uint64_t q0 = rowoff[i];
    const int64_t n = (int64_t)(rowoff[i + 1] - q0);
    uint64_t* g = keys + q0;
    // rank through bitmaps when that is cheaper than the bitonic network:
    // windows x (bitmap words + 2 key passes) vs npad log2(npad)^2 / 2 CAS
    int lg = 0;
    while ((1ll << lg) < n) lg++;
    const int64_t windows = (n_right + kRankWindow - 1) / kRankWindow;
    const bool rank = n > kSortBigCap ||
                      windows * ((int64_t)kRankWords / 2 + 6 * n) < (1ll << lg) * lg * (lg + 1);
    if (!rank) {
      for (int t = threadIdx.x; t < n; t += blockDim.x) sbuf[t] = g[t];
      __syncthreads();
      smem_bitonic<false>(sbuf, (int)n, threadIdx.x, blockDim.x);
      write_row(left_base + i, sbuf, q0, (int)n, threadIdx.x, blockDim.x, lefts, rights, sims);
      __syncthreads();
      continue;
    }
    uint32_t* bits = reinterpret_cast<uint32_t*>(sbuf);
    if (n <= (int64_t)kRankBatch * kSortBigThreads)
      rank_row<true>(g, n, q0, left_base + i, n_right, bits, bits + kRankWords, lefts, rights, sims);
    else
      rank_row<false>(g, n, q0, left_base + i, n_right, bits, bits + kRankWords, lefts, rights, sims);
  }
}

// ------------------------------------------------------ dense API kernels
// out[i*ldo + j] = canonical dot(left row i, bt column j); bt is the packed
// transpose (dim x nr, row stride ldb) exactly as sj_tile_dot takes it.
constexpr int kTD = 64, kTDK = 16;
__global__ void __launch_bounds__(256)
tile_dot_kernel(const float* __restrict__ left, int64_t lda, const float* __restrict__ bt,
                int64_t ldb, int64_t nl, int64_t nr, int dim, float* __restrict__ out,
                int64_t ldo) {
  __shared__ float As[kTDK][kTD + 1];
  __shared__ float Bs[kTDK][kTD];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = (int64_t)blockIdx.y * kTD, j0 = (int64_t)blockIdx.x * kTD;
  float acc[4][4] = {};
  for (int d0 = 0; d0 < dim; d0 += kTDK) {
    for (int e = threadIdx.x; e < kTD * kTDK; e += 256) {
      const int r = e / kTDK, d = e % kTDK;
      As[d][r] = (i0 + r < nl && d0 + d < dim) ? left[(i0 + r) * lda + d0 + d] : 0.0f;
      const int dd = e / kTD, c = e % kTD;
      Bs[dd][c] = (j0 + c < nr && d0 + dd < dim) ? bt[(int64_t)(d0 + dd) * ldb + j0 + c] : 0.0f;
    }
    __syncthreads();
    const int dm = min(kTDK, dim - d0);
    for (int d = 0; d < dm; d++) {
      float a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        a[u] = As[d][ty * 4 + u];
        b[u] = Bs[d][tx * 4 + u];
      }
#pragma unroll
      for (int u = 0; u < 4; u++)
#pragma unroll
        for (int w = 0; w < 4; w++) acc[u][w] = __fmaf_rn(a[u], b[w], acc[u][w]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; u++)
#pragma unroll
    for (int w = 0; w < 4; w++) {
      const int64_t i = i0 + ty * 4 + u, j = j0 + tx * 4 + w;
      if (i < nl && j < nr) out[i * ldo + j] = acc[u][w];
    }
}

// cosine_vm (linalg.py:70-84): out[i] = dot(a, m_i) / (||a|| * ||m_i||) with
// the reference's arithmetic -- sequential fmaf dot (sj_dots_vm), norms as
// fp64 sequential sums rounded to fp32 (sj_row_norms), then one fp32 multiply
// and one fp32 divide (numpy float32 ufuncs, round to nearest).  flags bit 0:
// ||a|| == 0, bit 1: some ||m_i|| == 0 (the reference raises ZeroVector).
// dots_vm (sj_dots_vm, _kernelcore.c:108-111) is the same kernel without the
// norms.
__device__ __forceinline__ float row_norm_dev(const float* x, int dim) {
  double ss = 0.0;
#pragma unroll 8
  for (int d = 0; d < dim; d++) {
    const double v = (double)x[d];
    ss = __fma_rn(v, v, ss);
  }
  return __double2float_rn(sqrt(ss));
}

// Persistent CTAs of 4 warps.  A warp owns 32 rows at a time and walks them
// in 32-column chunks; its (row group, chunk) items stream through two shared
// tiles with cp.async (item i+1 in flight while item i is consumed), every
// global load a coalesced row segment (16-byte copies when the rows allow).
// Lane r advances row r's chains -- the fp32 fmaf dot and the fp64 sum of
// squares -- over the chunk in column order, reading its row and the probe's
// chunk as 128-bit shared loads (pitch 36: conflict-free), so the arithmetic
// is exactly one-row-per-thread's.  The square of an fp32 value is exact in
// fp64, so dadd(ss, dmul(v, v)) == fma(v, v, ss): one DFMA per element.
constexpr int kVmWarps = 4;
constexpr int kVmPitch = 36;

__device__ __forceinline__ void vm_cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void vm_cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

template <bool kCos>
__device__ __forceinline__ void vm_step(float& acc, double& ss, float ak, float x) {
  acc = __fmaf_rn(ak, x, acc);
  if (kCos) {
    const double v = (double)x;
    ss = __fma_rn(v, v, ss);
  }
}

template <bool kCos>
__global__ void __launch_bounds__(kVmWarps * 32)
vm_rows_kernel(const float* __restrict__ a, const float* __restrict__ m, int64_t n, int dim,
               float* __restrict__ out, int* __restrict__ flags) {
  __shared__ __align__(16) float tile[kVmWarps][2][32][kVmPitch];
  __shared__ __align__(16) float ash[kVmWarps][2][32];
  __shared__ float na_s;
  __shared__ volatile int na_ready;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (kCos) {
    if (threadIdx.x == 0) na_ready = 0;
    __syncthreads();
    // the probe norm is a sequential chain: thread 0 runs it while the other
    // warps start streaming; they wait for it only before their first write
    if (threadIdx.x == 0) {
      na_s = row_norm_dev(a, dim);
      if (blockIdx.x == 0 && na_s == 0.0f) atomicOr(flags, 1);
      __threadfence_block();
      na_ready = 1;
    }
  }
  bool have_na = false;
  const int64_t groups = (n + 31) / 32;
  const int64_t gstride = (int64_t)gridDim.x * kVmWarps;
  const int nch = (dim + 31) / 32;
  const bool vec = (dim & 3) == 0 && ((reinterpret_cast<uintptr_t>(a) |
                                       reinterpret_cast<uintptr_t>(m)) & 15) == 0;
  auto issue = [&](int64_t g, int c, int b) {
    if (g < groups) {
      const int64_t r0 = g * 32;
      const int rows = (int)mn<int64_t>(32, n - r0);
      const int c0 = c * 32;
      if (vec) {
        const int q = lane & 7;
        if (c0 + 4 * q < dim) {
          const float* src = m + r0 * dim + c0 + 4 * q;
          for (int r = lane >> 3; r < rows; r += 4)
            vm_cp_async16(&tile[warp][b][r][4 * q], src + (int64_t)r * dim);
          if (lane < 8) vm_cp_async16(&ash[warp][b][4 * q], a + c0 + 4 * q);
        }
      } else if (c0 + lane < dim) {
        const float* src = m + r0 * dim + c0 + lane;
        for (int r = 0; r < rows; r++) vm_cp_async4(&tile[warp][b][r][lane], src + (int64_t)r * dim);
        vm_cp_async4(&ash[warp][b][lane], a + c0 + lane);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t g = (int64_t)blockIdx.x * kVmWarps + warp;
  int c = 0, b = 0;
  issue(g, 0, 0);
  float acc = 0.0f;
  double ss = 0.0;
  while (g < groups) {
    int64_t gn = g;
    int cn = c + 1;
    if (cn == nch) {
      cn = 0;
      gn = g + gstride;
    }
    issue(gn, cn, b ^ 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    const int cols = min(32, dim - c * 32);
    const float4* rw = reinterpret_cast<const float4*>(tile[warp][b][lane]);
    const float4* av = reinterpret_cast<const float4*>(ash[warp][b]);
    if (cols == 32) {
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const float4 x = rw[q], y = av[q];
        vm_step<kCos>(acc, ss, y.x, x.x);
        vm_step<kCos>(acc, ss, y.y, x.y);
        vm_step<kCos>(acc, ss, y.z, x.z);
        vm_step<kCos>(acc, ss, y.w, x.w);
      }
    } else {
      const float* rs = tile[warp][b][lane];
      const float* as = ash[warp][b];
      for (int k = 0; k < cols; k++) vm_step<kCos>(acc, ss, as[k], rs[k]);
    }
    __syncwarp();
    if (c == nch - 1) {
      const int64_t i = g * 32 + lane;
      if (i < n) {
        if (kCos) {
          if (!have_na) {
            while (na_ready == 0) {
            }
            __threadfence_block();
            have_na = true;
          }
          const float nr = __double2float_rn(sqrt(ss));
          if (nr == 0.0f) atomicOr(flags, 2);
          out[i] = __fdiv_rn(acc, __fmul_rn(na_s, nr));
        } else {
          out[i] = acc;
        }
      }
      acc = 0.0f;
      ss = 0.0;
    }
    g = gn;
    c = cn;
    b ^= 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Dense threshold scan, row-major order (sj_scan_count / sj_scan_fill).
__global__ void dense_count_kernel(const float* __restrict__ buf, int64_t nl, int64_t nr,
                                   float theta, uint32_t* __restrict__ rowcount) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= nl) return;
  uint32_t c = 0;
  for (int64_t j = lane; j < nr; j += 32) c += buf[i * nr + j] >= theta;
  c = __reduce_add_sync(0xffffffffu, c);
  if (lane == 0) rowcount[i] = c;
}

__global__ void dense_fill_kernel(const float* __restrict__ buf, int64_t nl, int64_t nr,
                                  float theta, const uint64_t* __restrict__ rowoff, uint64_t left0,
                                  uint64_t right0, uint64_t* __restrict__ lefts,
                                  uint64_t* __restrict__ rights, float* __restrict__ sims) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= nl) return;
  uint64_t q = rowoff[i];
  for (int64_t j0 = 0; j0 < nr; j0 += 32) {
    const int64_t j = j0 + lane;
    const float s = j < nr ? buf[i * nr + j] : 0.0f;
    const bool hit = j < nr && s >= theta;
    const unsigned b = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      const uint64_t pos = q + __popc(b & ((1u << lane) - 1u));
      lefts[pos] = left0 + (uint64_t)i;
      rights[pos] = right0 + (uint64_t)j;
      sims[pos] = s;
    }
    q += __popc(b);
  }
}

}  // namespace sjb
