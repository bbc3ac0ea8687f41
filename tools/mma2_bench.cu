// Microbenchmark: tcgen05.mma.cta_group::2 (M=256, kind::f16, SS) issue rate
// per CTA pair by N.  Leader lane 0 issues `iters` MMAs; reports cycles/MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma2_bench tools/mma2_bench.cu
#include <cstdio>
#include "../paper_2312_01476_b200/csrc/sjb_common.cuh"
using namespace sjb;

__device__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((addr & 0x3FFFF) >> 4);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  return d;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    bench2(int N, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 196 * 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 196 * 1024 + 8);
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t idesc = umma_idesc_bf16_f32(256, N);
  const uint32_t a_addr = smem_u32(smem), b_addr = a_addr + 64 * 1024;
  if (rank == 0 && threadIdx.x == 0) {
    const uint64_t ad0 = make_desc(a_addr, 2048, 128), bd0 = make_desc(b_addr, N * 8, 128);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 7) {
#pragma unroll
      for (int kk = 0; kk < 7; kk++) {
        uint64_t ad = ad0 + kk * (4096 >> 4), bd = bd0 + kk * ((N * 16) >> 4);
        uint32_t acc = (i | kk) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
    mbar_wait(bar, 0);
    out[blockIdx.x / 2] = (unsigned long long)(clock64() - t0);
  } else if (rank == 1 && threadIdx.x == 0) {
    mbar_wait(bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(bench2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 21000;
  for (int N : {64, 128, 256}) {
    bench2<<<148, 128, smem>>>(N, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h[74];
    cudaMemcpy(h, d, 74 * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 74; i++) mx = h[i] > mx ? h[i] : mx;
    printf("2CTA M=256 N=%3d: %.1f cyc/mma (floor %.0f)\n", N, mx / iters, 256.0 * N / 512.0);
  }
  return 0;
}
