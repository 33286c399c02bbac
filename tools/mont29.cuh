// Fr255 Montgomery product on 9 x 29-bit unsaturated limbs.
//
// Storage stays 8 x 32-bit Montgomery form with R = 2^256 (field.cuh).  On
// entry a is re-sliced into 29-bit limbs and b into 29-bit limbs of 32 b;
// the product runs operand-scanning Montgomery with radix 2^29 over 64-bit
// column accumulators, so every limb product is one IMAD.WIDE.U32 that
// accumulates in place (no add-with-carry chains):
//   a (32 b) 2^-261 = a b 2^-256 (mod p),
// i.e. the same Montgomery product as the 32-bit CIOS.  Bounds: limbs are
// < 2^29, so a limb product is < 2^58 and a column receives at most 9 a*b
// and 9 m*p products plus a carry < 2^35: < 2^63, no overflow.  With a, b < p
// the result is < a 32b / 2^261 + p < 1.5 p, so one conditional subtraction
// gives the canonical value.  p = 1 mod 2^29, hence n' = -p^-1 = -1 and
// m = -t0 mod 2^29; the m * p_0 product is an add.
#pragma once
#include <stdint.h>

namespace zkl {
namespace m29 {

constexpr uint32_t kMask = (1u << 29) - 1;

// bits [pos, pos + 29) of the 256-bit little-endian value v (pos may be < 0)
template <int POS>
ZKL_HD uint32_t limb(const uint32_t (&v)[8]) {
  if constexpr (POS < 0) {
    return (v[0] << (-POS)) & kMask;
  } else {
    constexpr int i = POS / 32, s = POS % 32;
    const uint32_t lo = v[i];
    const uint32_t hi = (i + 1 < 8) ? v[i + 1] : 0u;
    const uint64_t w = ((uint64_t)hi << 32) | lo;
    return (uint32_t)(w >> s) & kMask;
  }
}

template <int SHIFT>
ZKL_HD void split(const uint32_t (&v)[8], uint32_t (&x)[9]) {
  x[0] = limb<0 - SHIFT>(v);
  x[1] = limb<29 - SHIFT>(v);
  x[2] = limb<58 - SHIFT>(v);
  x[3] = limb<87 - SHIFT>(v);
  x[4] = limb<116 - SHIFT>(v);
  x[5] = limb<145 - SHIFT>(v);
  x[6] = limb<174 - SHIFT>(v);
  x[7] = limb<203 - SHIFT>(v);
  x[8] = limb<232 - SHIFT>(v);
}

// p in 29-bit limbs (p = 0x73EDA753...00000001)
ZKL_HD constexpr uint32_t kP(int j) {
  return j == 0 ? 0x00000001u : j == 1 ? 0x1ffffff8u : j == 2 ? 0x1f96ffbfu
       : j == 3 ? 0x1b4805ffu : j == 4 ? 0x1d80553bu : j == 5 ? 0x0c0404d0u
       : j == 6 ? 0x1520cce7u : j == 7 ? 0x0a6533afu : 0x0073eda7u;
}

// 9 normalised 29-bit limbs (value < 2^256) -> 8 x 32-bit words
ZKL_HD void join(const uint32_t (&l)[9], uint32_t (&v)[8]) {
  // word w covers bits [32w, 32w+32): limb k = floor(32w/29), s = 32w - 29k
  v[0] = l[0] | (l[1] << 29);
  v[1] = (l[1] >> 3) | (l[2] << 26);
  v[2] = (l[2] >> 6) | (l[3] << 23);
  v[3] = (l[3] >> 9) | (l[4] << 20);
  v[4] = (l[4] >> 12) | (l[5] << 17);
  v[5] = (l[5] >> 15) | (l[6] << 14);
  v[6] = (l[6] >> 18) | (l[7] << 11);
  v[7] = (l[7] >> 21) | (l[8] << 8);
}

// acc += a * b (u32 x u32 -> u64 accumulate: one IMAD.WIDE.U32)
ZKL_HD void mad(uint64_t& acc, uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
#else
  acc += (uint64_t)a * b;
#endif
}

// One Montgomery step: t += x * yi, then add m p (m = -t0 mod 2^29) and
// shift one limb.  t[k] are 64-bit column accumulators.
ZKL_HD void step(uint64_t (&t)[9], const uint32_t (&x)[9], uint32_t yi) {
#pragma unroll
  for (int j = 0; j < 9; j++) mad(t[j], x[j], yi);
  const uint32_t m = (0u - (uint32_t)t[0]) & kMask;
  const uint64_t c = (t[0] + m) >> 29;
#pragma unroll
  for (int j = 1; j < 9; j++) mad(t[j], m, kP(j));
#pragma unroll
  for (int j = 0; j < 8; j++) t[j] = t[j + 1];
  t[8] = 0;
  t[0] += c;
}

// r = a b 2^-256 mod p, a, b < p, 8 x 32-bit canonical Montgomery-form words
ZKL_HD void mul(const uint32_t (&a)[8], const uint32_t (&b)[8], uint32_t (&r)[8]) {
  uint32_t x[9], y[9];
  split<0>(a, x);
  split<5>(b, y);
  uint64_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < 9; i++) step(t, x, y[i]);
  uint32_t l[9];
#pragma unroll
  for (int j = 0; j < 8; j++) {
    l[j] = (uint32_t)t[j] & kMask;
    t[j + 1] += t[j] >> 29;
  }
  l[8] = (uint32_t)t[8];
  join(l, r);
}

}  // namespace m29
}  // namespace zkl
