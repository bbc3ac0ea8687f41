// sjb_fmt.cu -- the canonical matches file on the GPU: line i of the output
// is "<left>,<right>,<sim>\n" (the reference's cli._write_matches,
// cli.py:105-108), where <sim> is numpy's format_float_positional(
// float32(sim), unique=True, trim="-") (cli.py:99-102): the shortest decimal
// string that reads back as the same float32, printed without an exponent.
//
// The digits come from free-format Dragon4 (Steele & White's shortest
// digit generation with margins), restated in exact 192-bit integer
// arithmetic; the rounding-interval boundaries are inclusive when the float's
// mantissa is even (IEEE round-half-even on read-back), the variant numpy
// implements (pinned in oracle/fmt_oracle.py against numpy itself).
//
// Byte work: one thread per line, 256-line groups.
//   csv_layout_kernel  Dragon4 digits per line (kept, 12 B/line) and per-group
//                      byte counts (u32) -> run_scan -> u64 group offsets
//   csv_write_kernel   rebuild each line from its digits, block-scan the lengths,
//                      assemble the group's text in shared memory, store it
//                      coalesced.
#include "sjb_common.cuh"

namespace sjb {
namespace fmt {

constexpr int kLines = 256;    // lines per CTA (one per thread)
constexpr int kMaxLine = 91;   // 20 + 1 + 20 + 1 + 48 + 1

struct U192 {
  uint64_t w[3];
};

__device__ __forceinline__ U192 u192(uint64_t v) { return U192{{v, 0ull, 0ull}}; }

__device__ __forceinline__ U192 shl(uint64_t v, int s) {  // v << s, s < 128
  U192 r = u192(0);
  const int q = s >> 6, b = s & 63;
  r.w[q] = v << b;
  if (b && q + 1 < 3) r.w[q + 1] = v >> (64 - b);
  return r;
}

__device__ __forceinline__ void mul_small(U192& a, uint64_t k) {  // k < 2^32
  unsigned __int128 c = 0;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    c += (unsigned __int128)a.w[i] * k;
    a.w[i] = (uint64_t)c;
    c >>= 64;
  }
}

__device__ __forceinline__ void mul_pow10(U192& a, int k) {
  for (; k >= 9; k -= 9) mul_small(a, 1000000000ull);
  uint64_t p = 1;
  for (; k > 0; k--) p *= 10;
  if (p > 1) mul_small(a, p);
}

__device__ __forceinline__ int cmp(const U192& a, const U192& b) {
#pragma unroll
  for (int i = 2; i >= 0; i--)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}

__device__ __forceinline__ U192 add(const U192& a, const U192& b) {
  U192 r;
  unsigned __int128 c = 0;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    c += (unsigned __int128)a.w[i] + b.w[i];
    r.w[i] = (uint64_t)c;
    c >>= 64;
  }
  return r;
}

__device__ __forceinline__ void sub_in(U192& a, const U192& b) {  // a >= b
  uint64_t borrow = 0;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    const uint64_t x = a.w[i], y = b.w[i];
    const uint64_t d = x - y - borrow;
    borrow = (x < y || (x == y && borrow)) ? 1ull : 0ull;
    a.w[i] = d;
  }
}

// Shortest digits of a positive finite nonzero float32 (bits without sign):
// packed 4 bits per digit, first digit in the highest used nibble; returns the
// digit count, *exp10 = decimal exponent of the first digit.
__device__ int shortest_digits(uint32_t bits, uint64_t* packed, int* exp10) {
  const uint32_t be = (bits >> 23) & 0xFFu, f = bits & 0x7FFFFFu;
  uint64_t m;
  int ex, mbit;
  bool unequal;
  if (be) {
    m = f | (1u << 23);
    ex = (int)be - 150;
    mbit = 23;
    unequal = (f == 0 && be != 1);
  } else {
    m = f;
    ex = -149;
    mbit = 31 - __clz(f);
    unequal = false;
  }
  U192 val, scale, ml, mh;
  if (unequal) {
    if (ex > 0) {
      val = shl(4 * m, ex); scale = u192(4); ml = shl(1, ex); mh = shl(1, ex + 1);
    } else {
      val = u192(4 * m); scale = shl(1, -ex + 2); ml = u192(1); mh = u192(2);
    }
  } else {
    if (ex > 0) {
      val = shl(2 * m, ex); scale = u192(2); ml = shl(1, ex);
    } else {
      val = u192(2 * m); scale = shl(1, -ex + 1); ml = u192(1);
    }
    mh = ml;
  }
  // estimate of the first digit's exponent: exact or one too low
  int de = (int)ceil((double)(mbit + ex) * 0.30102999566398119521373889472449 - 0.69);
  if (de > 0) {
    mul_pow10(scale, de);
  } else if (de < 0) {
    mul_pow10(val, -de);
    mul_pow10(ml, -de);
    mh = ml;
    if (unequal) mh = add(ml, ml);
  }
  if (cmp(val, scale) >= 0) {
    de += 1;
  } else {
    mul_small(val, 10);
    mul_small(ml, 10);
    mh = unequal ? add(ml, ml) : ml;
  }
  *exp10 = de - 1;
  const bool incl = (m & 1) == 0;  // even mantissa: boundaries read back to it
  uint64_t digs = 0;
  int n = 0;
  uint32_t d;
  bool low, high;
  for (;;) {
    d = 0;
    while (cmp(val, scale) >= 0) {
      sub_in(val, scale);
      d++;
    }
    const U192 hi = add(val, mh);
    const int cl = cmp(val, ml), ch = cmp(hi, scale);
    low = incl ? cl <= 0 : cl < 0;
    high = incl ? ch >= 0 : ch > 0;
    if (low || high || n >= 16) break;
    digs = (digs << 4) | d;
    n++;
    mul_small(val, 10);
    mul_small(ml, 10);
    mh = unequal ? add(ml, ml) : ml;
  }
  bool round_down = low;
  if (low == high) {  // both or neither neighbour excluded: nearest digit, ties to even
    const U192 v2 = add(val, val);
    const int c = cmp(v2, scale);
    round_down = c < 0 || (c == 0 && (d & 1) == 0);
  }
  if (round_down) {
    digs = (digs << 4) | d;
    n++;
  } else if (d < 9) {
    digs = (digs << 4) | (d + 1);
    n++;
  } else {
    // carry through trailing nines of the digits already produced
    while (n > 0 && (digs & 0xF) == 9) {
      digs >>= 4;
      n--;
    }
    if (n == 0) {
      digs = 1;
      n = 1;
      *exp10 += 1;
    } else {
      digs += 1;
    }
  }
  *packed = digs;
  return n;
}

__device__ __forceinline__ int dec_len(uint64_t v) {
  int n = 1;
  while (v >= 10) {
    v /= 10;
    n++;
  }
  return n;
}

// The formatted pieces of one line.
struct Line {
  uint64_t l, r, digs;
  int nd, e10, len;
  uint32_t kind;  // 0 digits, 1 zero, 2 inf, 3 nan
  bool neg;
};

__device__ __forceinline__ int sim_len(const Line& s) {
  if (s.kind == 3) return 3;
  if (s.kind == 1) return 1 + s.neg;
  if (s.kind == 2) return 3 + s.neg;
  int body;
  if (s.e10 >= 0) body = s.nd <= s.e10 + 1 ? s.e10 + 1 : s.nd + 1;
  else body = 2 + (-s.e10 - 1) + s.nd;
  return body + s.neg;
}

// Per-line digits handed from the layout pass to the write pass (12 B/line),
// so Dragon4 runs once per line: packed digits, and nd | e10 | kind | sign.
__device__ __forceinline__ uint32_t pack_meta(const Line& s) {
  return (uint32_t)s.nd | ((uint32_t)(s.e10 + 128) << 8) | (s.kind << 16) |
         ((uint32_t)s.neg << 18);
}

__device__ __forceinline__ Line make_line(uint64_t l, uint64_t r, float sim) {
  Line s;
  s.l = l;
  s.r = r;
  const uint32_t b = __float_as_uint(sim);
  s.neg = (b >> 31) != 0;
  const uint32_t a = b & 0x7FFFFFFFu;
  s.nd = 0;
  s.e10 = 0;
  s.digs = 0;
  if (a == 0) s.kind = 1;
  else if (a == 0x7F800000u) s.kind = 2;
  else if (a > 0x7F800000u) { s.kind = 3; s.neg = false; }
  else {
    s.kind = 0;
    s.nd = shortest_digits(a, &s.digs, &s.e10);
  }
  s.len = dec_len(l) + 1 + dec_len(r) + 1 + sim_len(s) + 1;
  return s;
}

__device__ __forceinline__ Line unpack_line(uint64_t l, uint64_t r, uint64_t digs,
                                            uint32_t meta) {
  Line s;
  s.l = l;
  s.r = r;
  s.digs = digs;
  s.nd = (int)(meta & 0xFFu);
  s.e10 = (int)((meta >> 8) & 0xFFu) - 128;
  s.kind = (meta >> 16) & 3u;
  s.neg = ((meta >> 18) & 1u) != 0;
  s.len = dec_len(l) + 1 + dec_len(r) + 1 + sim_len(s) + 1;
  return s;
}

__device__ __forceinline__ char* put_dec(char* o, uint64_t v, int n) {
  for (int i = n - 1; i >= 0; i--) {
    o[i] = (char)('0' + v % 10);
    v /= 10;
  }
  return o + n;
}

__device__ void put_line(char* o, const Line& s) {
  o = put_dec(o, s.l, dec_len(s.l));
  *o++ = ',';
  o = put_dec(o, s.r, dec_len(s.r));
  *o++ = ',';
  if (s.neg) *o++ = '-';
  if (s.kind == 1) {
    *o++ = '0';
  } else if (s.kind == 2) {
    *o++ = 'i'; *o++ = 'n'; *o++ = 'f';
  } else if (s.kind == 3) {
    *o++ = 'n'; *o++ = 'a'; *o++ = 'n';
  } else {
    auto digit = [&](int i) { return (char)('0' + ((s.digs >> (4 * (s.nd - 1 - i))) & 0xF)); };
    if (s.e10 >= 0) {
      for (int i = 0; i <= s.e10; i++) *o++ = i < s.nd ? digit(i) : '0';
      if (s.nd > s.e10 + 1) {
        *o++ = '.';
        for (int i = s.e10 + 1; i < s.nd; i++) *o++ = digit(i);
      }
    } else {
      *o++ = '0';
      *o++ = '.';
      for (int i = 0; i < -s.e10 - 1; i++) *o++ = '0';
      for (int i = 0; i < s.nd; i++) *o++ = digit(i);
    }
  }
  *o = '\n';
}

__device__ __forceinline__ uint32_t block_sum_u32(uint32_t x, uint32_t* red) {
  x = __reduce_add_sync(0xffffffffu, x);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  uint32_t t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < kLines / 32 ? red[threadIdx.x] : 0u;
    t = __reduce_add_sync(0xffffffffu, t);
  }
  return t;  // valid in thread 0
}

__global__ void __launch_bounds__(kLines)
csv_layout_kernel(const uint64_t* __restrict__ lefts, const uint64_t* __restrict__ rights,
                  const float* __restrict__ sims, int64_t n, uint32_t* __restrict__ group_len,
                  uint64_t* __restrict__ digs, uint32_t* __restrict__ meta) {
  __shared__ uint32_t red[kLines / 32];
  const int64_t i = (int64_t)blockIdx.x * kLines + threadIdx.x;
  uint32_t len = 0;
  if (i < n) {
    const Line s = make_line(lefts[i], rights[i], sims[i]);
    len = (uint32_t)s.len;
    digs[i] = s.digs;
    meta[i] = pack_meta(s);
  }
  const uint32_t t = block_sum_u32(len, red);
  if (threadIdx.x == 0) group_len[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kLines)
csv_write_kernel(const uint64_t* __restrict__ lefts, const uint64_t* __restrict__ rights,
                 const uint64_t* __restrict__ digs, const uint32_t* __restrict__ meta, int64_t n,
                 const uint64_t* __restrict__ group_off, uint8_t* __restrict__ out) {
  __shared__ char text[kLines * kMaxLine];
  __shared__ uint32_t wsum[kLines / 32];
  const int64_t i = (int64_t)blockIdx.x * kLines + threadIdx.x;
  Line s;
  s.len = 0;
  if (i < n) s = unpack_line(lefts[i], rights[i], digs[i], meta[i]);
  // block exclusive scan of the line lengths
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = (uint32_t)s.len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t base = 0, total = 0;
#pragma unroll
  for (int k = 0; k < kLines / 32; k++) {
    const uint32_t x = wsum[k];
    base += k < w ? x : 0u;
    total += x;
  }
  if (i < n) put_line(text + base + incl - (uint32_t)s.len, s);
  __syncthreads();
  uint8_t* dst = out + group_off[blockIdx.x];
  for (uint32_t k = threadIdx.x; k < total; k += kLines) dst[k] = (uint8_t)text[k];
}

}  // namespace fmt
}  // namespace sjb
