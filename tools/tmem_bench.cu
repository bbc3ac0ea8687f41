// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM.
// nwarps warps (multiple of 4); warp w reads its lane quarter (w % 4), each
// load moves 32 lanes x X columns x 4 B.  Reports bytes/cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include "../paper_2312_01476_b200/csrc/sjb_common.cuh"

using namespace sjb;

#define LD64(taddr, v, o) asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];" \
  : "=f"(v[o+0]),"=f"(v[o+1]),"=f"(v[o+2]),"=f"(v[o+3]),"=f"(v[o+4]),"=f"(v[o+5]),"=f"(v[o+6]),"=f"(v[o+7]),"=f"(v[o+8]),"=f"(v[o+9]),"=f"(v[o+10]),"=f"(v[o+11]),"=f"(v[o+12]),"=f"(v[o+13]),"=f"(v[o+14]),"=f"(v[o+15]), \
    "=f"(v[o+16]),"=f"(v[o+17]),"=f"(v[o+18]),"=f"(v[o+19]),"=f"(v[o+20]),"=f"(v[o+21]),"=f"(v[o+22]),"=f"(v[o+23]),"=f"(v[o+24]),"=f"(v[o+25]),"=f"(v[o+26]),"=f"(v[o+27]),"=f"(v[o+28]),"=f"(v[o+29]),"=f"(v[o+30]),"=f"(v[o+31]), \
    "=f"(v[o+32]),"=f"(v[o+33]),"=f"(v[o+34]),"=f"(v[o+35]),"=f"(v[o+36]),"=f"(v[o+37]),"=f"(v[o+38]),"=f"(v[o+39]),"=f"(v[o+40]),"=f"(v[o+41]),"=f"(v[o+42]),"=f"(v[o+43]),"=f"(v[o+44]),"=f"(v[o+45]),"=f"(v[o+46]),"=f"(v[o+47]), \
    "=f"(v[o+48]),"=f"(v[o+49]),"=f"(v[o+50]),"=f"(v[o+51]),"=f"(v[o+52]),"=f"(v[o+53]),"=f"(v[o+54]),"=f"(v[o+55]),"=f"(v[o+56]),"=f"(v[o+57]),"=f"(v[o+58]),"=f"(v[o+59]),"=f"(v[o+60]),"=f"(v[o+61]),"=f"(v[o+62]),"=f"(v[o+63]) : "r"(taddr))

// one x64 load per wait
__global__ void bench64(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t q = warp & 3;
  const uint32_t colbase = (warp >> 2) * 64;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    float v[64];
    LD64(tmem + ((q * 32) << 16) + (colbase & 511), v, 0);
    tc_wait_ld();
#pragma unroll
    for (int k = 0; k < 64; k += 2) acc += v[k];
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
    const int iters = 4000;
    bench64<<<148, nw * 32>>>(iters, d, s);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
    printf("warps=%2d x64 single : %.1f B/cycle/SM (%.1f cycles per x64 per warp)\n", nw,
           (double)iters * nw * 32 * 64 * 4 / mx, mx / iters);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
