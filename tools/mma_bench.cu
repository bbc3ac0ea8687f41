// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, SS) issue throughput
// per SM for operand layouts / N.  One CTA per SM; one thread issues `iters`
// MMAs back to back into one TMEM accumulator, commits, waits.  Data is
// garbage; only the timing matters.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdlib>
#include "../paper_2312_01476_b200/csrc/sjb_common.cuh"

using namespace sjb;

__device__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((addr & 0x3FFFF) >> 4);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(layout & 7) << 61;
  return d;
}

// layout: 0 = no swizzle (core matrices [kgroup][rows][16B]), 6 = SW32, 2 = SW128
__global__ void __launch_bounds__(128, 1) bench(int layout, int N, int iters, int ksteps,
                                                unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t& bar = *reinterpret_cast<uint64_t*>(smem + 196 * 1024);
  uint32_t& tslot = *reinterpret_cast<uint32_t*>(smem + 196 * 1024 + 8);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t a_addr = smem_u32(smem);
  const uint32_t b_addr = a_addr + 64 * 1024;
  const uint32_t idesc = umma_idesc_bf16_f32(128, N);
  if (threadIdx.x == 0) {
    // precomputed descriptors; per k-step only the 14-bit start address moves
    uint64_t ad0, bd0;
    uint32_t astep, bstep;  // encoded (16 B units) advance per k-step
    if (layout == 0) {
      ad0 = make_desc(a_addr, 2048, 128, 0);
      bd0 = make_desc(b_addr, N * 16, 128, 0);
      astep = 4096 >> 4;
      bstep = (N * 32) >> 4;
    } else if (layout == 6) {
      ad0 = make_desc(a_addr, 16, 256, 6);
      bd0 = make_desc(b_addr, 16, 256, 6);
      astep = 4096 >> 4;
      bstep = (N * 32) >> 4;
    } else {
      ad0 = make_desc(a_addr, 16, 1024, 2);
      bd0 = make_desc(b_addr, 16, 1024, 2);
      astep = 32 >> 4;  // within one atom (ignore atom crossing for timing)
      bstep = 32 >> 4;
    }
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 7) {
#pragma unroll
      for (int kk = 0; kk < 7; kk++)
        tc_mma_bf16(tmem, ad0 + kk * astep, bd0 + kk * bstep, idesc, (i | kk) ? 1u : 0u);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 21000;
  int layouts[3] = {0, 6, 2};
  const char* names[3] = {"noswz", "sw32", "sw128"};
  int Ns[3] = {64, 128, 256};
  for (int li = 0; li < 3; li++)
    for (int ni = 0; ni < 3; ni++) {
      const int N = Ns[ni];
      for (int grid : {1, sms}) {
        bench<<<grid, 128, smem>>>(layouts[li], N, iters, 7, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        unsigned long long h[256];
        cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < grid; i++) mx = h[i] > mx ? h[i] : mx;
        const double ideal = 128.0 * N / 256.0;
        printf("%-6s N=%3d grid=%3d: %.1f cyc/mma (floor %.0f) -> %.0f%% of floor\n", names[li],
               N, grid, mx / iters, ideal, 100.0 * ideal / (mx / iters));
      }
    }
  return 0;
}
