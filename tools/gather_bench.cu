// Microbenchmark: ways to feed the dense recheck's canonical chains with
// randomly indexed fp32 S rows (d = 100) -- the cfg5 theta = 0.4 access
// pattern (one R row per ~400 consecutive candidates, random S rows).
//   0 direct   per-lane 32-byte loads (recheck_grouped_kernel)
//   1 lanes    per-lane 1-D bulk copies (compiler waterfall over lanes)
//   2 lane0    lane 0 issues the warp's 32 1-D bulk copies (shuffled indices)
//   3 g4       lane 0 issues 8 tile::gather4 tensor copies, groups 1600 B apart
//              (faults: the destination of a tensor copy must be 128-byte aligned)
//   4 g4a      the same, groups 128-byte aligned (1664 B apart)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/gather_bench tools/gather_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int D = 100, NQ = D / 4, W = 7;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}"
               ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void g4(void* dst, const CUtensorMap* m, int c, int r0, int r1, int r2, int r3,
                                   uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               ::"r"(su32(dst)), "l"(m), "r"(c), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(b)) : "memory");
}

// candidates k: row i = k / per_row, right offset js[k]
__global__ void direct_kernel(const uint32_t* js, int64_t n, int per_row, const float* l32,
                              const float* r32, float* out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const float4* a = reinterpret_cast<const float4*>(l32 + (k / per_row) * D);
    const float4* b = reinterpret_cast<const float4*>(r32 + (size_t)js[k] * D);
    float x = 0.f;
#pragma unroll 5
    for (int q = 0; q < NQ; q++) {
      const float4 p = __ldg(a + q), s = __ldg(b + q);
      x = __fmaf_rn(p.x, s.x, x); x = __fmaf_rn(p.y, s.y, x);
      x = __fmaf_rn(p.z, s.z, x); x = __fmaf_rn(p.w, s.w, x);
    }
    out[k] = x;
  }
}

template <int MODE>
__global__ void __launch_bounds__(W * 32, 1)
staged_kernel(const uint32_t* js, int64_t n, int per_row, const float* l32, const float* r32,
              float* out, const __grid_constant__ CUtensorMap tmap, unsigned* work) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gstride = MODE == 4 ? 1664 : 1600;           // bytes per 4-row group
  const int bufbytes = 8 * gstride;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + 2 * warp;
  uint8_t* stage = sm + 128 + (size_t)warp * 2 * bufbytes;
  if (lane == 0) { mbar_init(bar, 1); mbar_init(bar + 1, 1); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t phase = 0;
  const int64_t nb_all = (n + 31) / 32;
  // lane p's row inside a buffer
  auto rowp = [&](int buf, int p) -> const float* {
    return reinterpret_cast<const float*>(stage + buf * bufbytes + (p >> 2) * gstride + (p & 3) * 400);
  };
  auto issue = [&](int64_t b, int buf) -> uint32_t {
    const int64_t k = b * 32 + lane;
    const uint32_t j = k < n ? js[k] : 0u;
    const uint32_t cnt = (uint32_t)(n - b * 32 < 32 ? n - b * 32 : 32);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (MODE == 1) {
      if (lane == 0) mbar_expect(bar + buf, cnt * 400);
      __syncwarp();
      if (k < n) bulk((void*)rowp(buf, lane), r32 + (size_t)j * D, 400, bar + buf);
    } else if (MODE == 2) {
      if (lane == 0) mbar_expect(bar + buf, cnt * 400);
      for (int r = 0; r < 32; r++) {
        const uint32_t jr = __shfl_sync(0xffffffffu, j, r);
        if (lane == 0 && r < (int)cnt) bulk((void*)rowp(buf, r), r32 + (size_t)jr * D, 400, bar + buf);
      }
    } else {
      const int groups = (int)((cnt + 3) / 4);
      if (lane == 0) mbar_expect(bar + buf, groups * 1600);
      for (int g = 0; g < 8; g++) {
        const uint32_t j0 = __shfl_sync(0xffffffffu, j, 4 * g), j1 = __shfl_sync(0xffffffffu, j, 4 * g + 1);
        const uint32_t j2 = __shfl_sync(0xffffffffu, j, 4 * g + 2), j3 = __shfl_sync(0xffffffffu, j, 4 * g + 3);
        if (lane == 0 && g < groups)
          g4((void*)rowp(buf, 4 * g), &tmap, 0, (int)j0, (int)j1, (int)j2, (int)j3, bar + buf);
      }
    }
    return j;
  };
  for (;;) {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(work, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    // a chunk = 13 batches (one R row's ~400 candidates)
    const int64_t b0 = (int64_t)c * 13;
    if (b0 >= nb_all) break;
    const int64_t b1 = (b0 + 13 < nb_all ? b0 + 13 : nb_all);
    uint32_t jc = issue(b0, (int)(b0 & 1));
    for (int64_t b = b0; b < b1; b++) {
      const int buf = (int)(b & 1);
      const uint32_t jn = b + 1 < b1 ? issue(b + 1, buf ^ 1) : 0u;
      mbar_wait(bar + buf, (phase >> buf) & 1u);
      phase ^= 1u << buf;
      const int64_t k = b * 32 + lane;
      if (k < n) {
        const float4* a = reinterpret_cast<const float4*>(l32 + (k / per_row) * D);
        const float4* s4 = reinterpret_cast<const float4*>(rowp(buf, lane));
        float x = 0.f;
#pragma unroll 5
        for (int q = 0; q < NQ; q++) {
          const float4 p = __ldg(a + q), s = s4[q];
          x = __fmaf_rn(p.x, s.x, x); x = __fmaf_rn(p.y, s.y, x);
          x = __fmaf_rn(p.z, s.z, x); x = __fmaf_rn(p.w, s.w, x);
        }
        out[k] = x;
      }
      jc = jn;
    }
    (void)jc;
  }
}

int main(int argc, char** argv) {
  const int64_t nS = 200000, nL = 200000, per_row = 400;
  const int64_t n = argc > 1 ? atoll(argv[1]) : 80000000;
  std::vector<float> hs(nS * D), hl(nL * D);
  srand(1);
  for (auto& v : hs) v = (rand() / (float)RAND_MAX) - 0.5f;
  for (auto& v : hl) v = (rand() / (float)RAND_MAX) - 0.5f;
  std::vector<uint32_t> hj(n);
  for (int64_t k = 0; k < n; k++) hj[k] = (uint32_t)(((uint64_t)rand() * 7919u + k) % nS);
  float *dS, *dL, *o0, *o1;
  uint32_t* dj;
  unsigned* work;
  CK(cudaMalloc(&dS, nS * D * 4)); CK(cudaMalloc(&dL, nL * D * 4));
  CK(cudaMalloc(&o0, n * 4)); CK(cudaMalloc(&o1, n * 4)); CK(cudaMalloc(&dj, n * 4));
  CK(cudaMalloc(&work, 4));
  CK(cudaMemcpy(dS, hs.data(), nS * D * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dL, hl.data(), nL * D * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dj, hj.data(), n * 4, cudaMemcpyHostToDevice));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {D, (cuuint64_t)nS};
  const cuuint64_t strides[1] = {D * 4};
  const cuuint32_t box[2] = {D, 1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dS, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc %d\n", (int)r);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int smem = 128 + W * 2 * 8 * 1664;
  auto run = [&](int mode, float* out) {
    CK(cudaMemset(work, 0, 4));
    if (mode == 0) direct_kernel<<<sms * 8, 256>>>(dj, n, per_row, dL, dS, out);
    else if (mode == 1) staged_kernel<1><<<sms, W * 32, smem>>>(dj, n, per_row, dL, dS, out, tm, work);
    else if (mode == 2) staged_kernel<2><<<sms, W * 32, smem>>>(dj, n, per_row, dL, dS, out, tm, work);
    else if (mode == 3) staged_kernel<3><<<sms, W * 32, smem>>>(dj, n, per_row, dL, dS, out, tm, work);
    else staged_kernel<4><<<sms, W * 32, smem>>>(dj, n, per_row, dL, dS, out, tm, work);
  };
  CK(cudaFuncSetAttribute(staged_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(staged_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(staged_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(staged_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  run(0, o0);
  CK(cudaDeviceSynchronize());
  std::vector<uint32_t> ref(n), got(n);
  CK(cudaMemcpy(ref.data(), o0, n * 4, cudaMemcpyDeviceToHost));
  const char* names[] = {"direct", "lanes", "lane0", "g4", "g4a"};
  const char* modes = argc > 2 ? argv[2] : "0124";
  for (const char* mp = modes; *mp; mp++) {
    const int mode = *mp - '0';
    CK(cudaMemset(o1, 0, n * 4));
    run(mode, o1);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("%s: error %s\n", names[mode], cudaGetErrorString(err)); return 1; }
    CK(cudaMemcpy(got.data(), o1, n * 4, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t k = 0; k < n; k++) bad += got[k] != ref[k];
    float best = 1e9f;
    for (int it = 0; it < 5; it++) {
      CK(cudaEventRecord(e0));
      run(mode, o1);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf("%-7s %8.3f ms  %.2f Grows/s  %.2f TB/s of S rows  mismatches %lld\n", names[mode], best,
           n / best / 1e6, n * 400.0 / best / 1e9, (long long)bad);
  }
  return 0;
}
