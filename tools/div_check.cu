// Brute-force check of the hoisted-reciprocal quotient used by
// normalize_row_smem (sjb_prep.cu) against __ddiv_rn: x float (all
// exponents), norm a double >= 1e-12 (random, near powers of two, and
// all-ones mantissas).  Reports mismatches in the double quotient and in the
// final float.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cmath>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void check(uint64_t seed, uint64_t per_thread, unsigned long long* bad64,
                      unsigned long long* bad32) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long b64 = 0, b32 = 0;
  for (uint64_t i = 0; i < per_thread; i++) {
    const uint64_t z = mix(seed ^ (t * per_thread + i) * 0xD1B54A32D192ED03ULL);
    const uint64_t w = mix(z);
    double norm;
    switch (w & 3) {
      case 0:  // random mantissa, exponent in [-40, 64]
        norm = __longlong_as_double((long long)(((uint64_t)(1023 - 40 + (w >> 8) % 105) << 52) |
                                                (z & 0xFFFFFFFFFFFFFULL)));
        break;
      case 1:  // mantissa near all-ones
        norm = __longlong_as_double((long long)(((uint64_t)(1023 + (w >> 8) % 8) << 52) |
                                                (0xFFFFFFFFFFFFFULL - (z & 0xFFFF))));
        break;
      case 2:  // mantissa near 1.0
        norm = __longlong_as_double((long long)(((uint64_t)(1023 + (w >> 8) % 8) << 52) |
                                                (z & 0xFFFF)));
        break;
      default:  // sqrt of a random sum of squares, the production distribution
        norm = sqrt(__longlong_as_double((long long)(((uint64_t)(1013 + (w >> 8) % 30) << 52) |
                                                     (z & 0xFFFFFFFFFFFFFULL))));
    }
    if (norm < 1e-12) norm = 1e-12;
    const uint32_t xb = (uint32_t)(z >> 20) & 0x7FFFFFFFu;
    float xf = __uint_as_float((w >> 40) & 1 ? xb : (xb & 0x807FFFFFu) | (((uint32_t)(w >> 44) % 20 + 117u) << 23));
    if (!isfinite(xf)) xf = 1.0f;
    if ((w >> 50) & 1) xf = -xf;
    const double x = (double)xf;
    const double ref = __ddiv_rn(x, norm);
    const double y = __drcp_rn(norm);
    const double q0 = __dmul_rn(x, y);
    const double q = copysign(__fma_rn(__fma_rn(-q0, norm, x), y, q0), x);
    if (__double_as_longlong(q) != __double_as_longlong(ref) && b64 < 2)
      printf("x=%a norm=%a ref=%a q=%a q0=%a y=%a case=%d\n", x, norm, ref, q, q0, y, (int)(w & 3));
    b64 += (__double_as_longlong(q) != __double_as_longlong(ref));
    b32 += (__float_as_uint(__double2float_rn(q)) != __float_as_uint(__double2float_rn(ref)));
  }
  if (b64) atomicAdd(bad64, b64);
  if (b32) atomicAdd(bad32, b32);
}

int main(int argc, char** argv) {
  const int rounds = argc > 1 ? atoi(argv[1]) : 16;
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  const int blocks = 148 * 16, threads = 256;
  const uint64_t per = 1 << 12;
  for (int r = 0; r < rounds; r++) check<<<blocks, threads>>>(0x1234 + r * 977ULL, per, d, d + 1);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double total = (double)rounds * blocks * threads * per;
  printf("trials %.3e  double mismatches %llu  float mismatches %llu  err %s\n", total, h[0], h[1],
         cudaGetErrorString(cudaGetLastError()));
  return h[0] || h[1];
}
