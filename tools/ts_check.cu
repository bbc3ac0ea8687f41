// ts_check.cu -- does tcgen05.mma with A in tensor memory (loaded from the
// filter's shared-memory operand layout by tcgen05.cp.128x256b) give the same
// accumulators as the SS-mode MMA the filter uses?  One CTA, M=128, N=128,
// K=112 (7 k-steps), fp16 inputs, fp32 accumulate.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o tools/bin/ts_check tools/ts_check.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
#include "../paper_2312_01476_b200/csrc/sjb_common.cuh"

using namespace sjb;

constexpr int KP = 112, KS = KP / 16, ROWS = 256;

__device__ __forceinline__ void tc_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void tc_mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b_desc,
                                          uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

// A, B: operand images [KP/8][256][8] fp16 (the filter's tile layout).
__global__ void k(const __half* A, const __half* B, float* out_ss, float* out_ts, int half) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;
  uint8_t* sb = sm + ROWS * KP * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + ROWS * KP * 2);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < ROWS * KP / 8; i += blockDim.x) {
    reinterpret_cast<uint4*>(sa)[i] = reinterpret_cast<const uint4*>(A)[i];
    reinterpret_cast<uint4*>(sb)[i] = reinterpret_cast<const uint4*>(B)[i];
  }
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *slot;
  const uint32_t lbo = ROWS * 16, sbo = 128;
  const uint64_t kstep = (2 * lbo) >> 4;
  const uint64_t ad = umma_desc_kmajor_noswz(smem_u32(sa), lbo, sbo) + half * ((128 * 16) >> 4);
  const uint64_t bd = umma_desc_kmajor_noswz(smem_u32(sb), lbo, sbo);
  const uint32_t idesc = umma_idesc_f16_f32(128, 128);
  if (warp == 0) {
    // SS into columns 0..127; A copied to columns 256.. (8 per k-step); TS into 128..255
    for (int kk = 0; kk < KS; kk++) tc_mma_f16_elect(tm, ad + kk * kstep, bd + kk * kstep, idesc, kk > 0);
    if (lane == 0) {
      for (int kk = 0; kk < KS; kk++) tc_cp_128x256b(tm + 256 + kk * 8, ad + kk * kstep);
      for (int kk = 0; kk < KS; kk++) tc_mma_ts(tm + 128, tm + 256 + kk * 8, bd + kk * kstep, idesc, kk > 0);
    }
    tc_commit_elect(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  if (warp < 4) {
    float v[64];
    for (int which = 0; which < 2; which++)
      for (int c = 0; c < 2; c++) {
        SJB_TMEM_LD64(tm + ((warp * 32) << 16) + which * 128 + c * 64, v);
        tc_wait_ld();
        float* o = which ? out_ts : out_ss;
        for (int j = 0; j < 64; j++) o[(warp * 32 + lane) * 128 + c * 64 + j] = v[j];
      }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

int main() {
  const int n = ROWS * KP;
  __half *hA = (__half*)malloc(n * 2), *hB = (__half*)malloc(n * 2);
  float* a = (float*)malloc(n * 4);
  float* b = (float*)malloc(n * 4);
  srand(1);
  // logical X[r][k] stored at [(k/8)*ROWS + r]*8 + k%8
  for (int r = 0; r < ROWS; r++)
    for (int kk = 0; kk < KP; kk++) {
      const float x = (rand() % 2001 - 1000) / 1024.0f, y = (rand() % 2001 - 1000) / 1024.0f;
      const int idx = ((kk / 8) * ROWS + r) * 8 + kk % 8;
      hA[idx] = __float2half(x); hB[idx] = __float2half(y);
      a[r * KP + kk] = __half2float(hA[idx]); b[r * KP + kk] = __half2float(hB[idx]);
    }
  __half *dA, *dB; float *dss, *dts;
  cudaMalloc(&dA, n * 2); cudaMalloc(&dB, n * 2);
  cudaMalloc(&dss, 128 * 128 * 4); cudaMalloc(&dts, 128 * 128 * 4);
  cudaMemcpy(dA, hA, n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, n * 2, cudaMemcpyHostToDevice);
  const int smem = 2 * ROWS * KP * 2 + 64;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int bad = 0;
  for (int half = 0; half < 2; half++) {
    k<<<1, 128, smem>>>(dA, dB, dss, dts, half);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    float *ss = (float*)malloc(128 * 128 * 4), *ts = (float*)malloc(128 * 128 * 4);
    cudaMemcpy(ss, dss, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ts, dts, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    double maxref = 0, maxdiff_ts = 0;
    int neq = 0;
    for (int i = 0; i < 128; i++)
      for (int j = 0; j < 128; j++) {
        double r = 0;
        for (int kk = 0; kk < KP; kk++) r += (double)a[(half * 128 + i) * KP + kk] * b[j * KP + kk];
        maxref = fmax(maxref, fabs(ss[i * 128 + j] - r));
        maxdiff_ts = fmax(maxdiff_ts, fabs(ts[i * 128 + j] - ss[i * 128 + j]));
        neq += ts[i * 128 + j] != ss[i * 128 + j];
      }
    printf("half %d: |SS - fp64 ref| max %.3g   |TS - SS| max %.3g  (%d of 16384 differ)\n", half,
           maxref, maxdiff_ts, neq);
    bad += maxref > 1e-3 || neq != 0;
  }
  printf(bad ? "TS MISMATCH\n" : "TS OK\n");
  return bad;
}
