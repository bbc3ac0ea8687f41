// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM.
// nwarps warps (multiple of 4); warp w reads its lane quarter (w % 4), each
// load moves 32 lanes x X columns x 4 B.  Reports bytes/cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include "../paper_2312_01476_b200/csrc/sjb_common.cuh"

using namespace sjb;

template <int CHUNKS>  // x32 loads per wait
__global__ void bench(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t q = warp & 3;
  const uint32_t colbase = (warp >> 2) * 128;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    float v[32 * CHUNKS];
#pragma unroll
    for (int c = 0; c < CHUNKS; c++) {
      const uint32_t taddr = tmem + ((q * 32) << 16) + ((colbase + c * 32) & 511);
      SJB_TMEM_LD32(taddr, v, c * 32);
    }
    tc_wait_ld();
#pragma unroll
    for (int k = 0; k < 32 * CHUNKS; k += 2) acc += v[k];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 12345.f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int CHUNKS>
void run(int nwarps, unsigned long long* d, float* s) {
  const int iters = 4000;
  bench<CHUNKS><<<148, nwarps * 32>>>(iters, d, s);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  const double bytes = (double)iters * nwarps * 32 * 32 * CHUNKS * 4;
  printf("warps=%2d chunks/wait=%d : %.1f B/cycle/SM (%.1f cycles per x32 per warp)\n", nwarps,
         CHUNKS, bytes / mx, mx / (iters * CHUNKS));
}

int main() {
  unsigned long long* d;
  float* s;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&s, 4);
  for (int nw : {4, 8, 16}) {
    run<1>(nw, d, s);
    run<2>(nw, d, s);
    run<4>(nw, d, s);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
