// Host-side scalar field arithmetic for the drivers (transcript-side work:
// challenges, term coefficients, round-evaluation finishing).
//
// Same element layout as the device (field.cuh): Fr255 values are 32-byte
// little-endian Montgomery residues (R = 2^256), M61 values canonical u64.
// Fr255 here uses 4 x 64-bit limbs with 128-bit products (CIOS), ~8x fewer
// multiply instructions than the portable 32-bit-limb code in field.cuh.
#pragma once
#include <stdint.h>
#include <string.h>

#include "field.cuh"

namespace zkl {
namespace host {

using u128 = unsigned __int128;

struct Fr {
  using T = fr_t;
  static constexpr uint64_t P[4] = {0xffffffff00000001ull, 0x53bda402fffe5bfeull,
                                    0x3339d80809a1d805ull, 0x73eda753299d7d48ull};
  static constexpr uint64_t NINV = 0xfffffffeffffffffull;  // -p^-1 mod 2^64
  static constexpr uint64_t R2[4] = {0xc999e990f3f29c6dull, 0x2b6cedcb87925c23ull,
                                     0x05d314967254398full, 0x0748d9d99f59ff11ull};

  static inline void ld(const T& a, uint64_t (&x)[4]) { memcpy(x, &a, 32); }
  static inline T st(const uint64_t (&x)[4]) {
    T r;
    memcpy(&r, x, 32);
    return r;
  }
  static inline bool geq_p(const uint64_t (&x)[4]) {
    for (int i = 3; i >= 0; i--) {
      if (x[i] != P[i]) return x[i] > P[i];
    }
    return true;
  }
  static inline void sub_p(uint64_t (&x)[4]) {
    u128 br = 0;
    for (int i = 0; i < 4; i++) {
      u128 d = (u128)x[i] - P[i] - br;
      x[i] = (uint64_t)d;
      br = (d >> 64) & 1;
    }
  }
  static inline T add(const T& a, const T& b) {
    uint64_t x[4], y[4];
    ld(a, x);
    ld(b, y);
    u128 c = 0;
    for (int i = 0; i < 4; i++) {
      c += (u128)x[i] + y[i];
      x[i] = (uint64_t)c;
      c >>= 64;
    }
    if (geq_p(x)) sub_p(x);  // a + b < 2p < 2^256
    return st(x);
  }
  static inline T sub(const T& a, const T& b) {
    uint64_t x[4], y[4];
    ld(a, x);
    ld(b, y);
    u128 br = 0;
    for (int i = 0; i < 4; i++) {
      u128 d = (u128)x[i] - y[i] - br;
      x[i] = (uint64_t)d;
      br = (d >> 64) & 1;
    }
    if (br) {
      u128 c = 0;
      for (int i = 0; i < 4; i++) {
        c += (u128)x[i] + P[i];
        x[i] = (uint64_t)c;
        c >>= 64;
      }
    }
    return st(x);
  }
  // Montgomery product a * b / 2^256 mod p (inputs < p)
  static inline T mul(const T& a, const T& b) {
#if defined(__x86_64__) && !defined(__CUDA_ARCH__)
    if (has_adx()) return mul_adx(a, b);
#endif
    return mul_portable(a, b);
  }
#if defined(__x86_64__) && !defined(__CUDA_ARCH__)
  static inline bool has_adx() {
    static const bool v = __builtin_cpu_supports("adx") && __builtin_cpu_supports("bmi2");
    return v;
  }
  // the same CIOS product with MULX and the two carry chains of ADCX / ADOX
  // (CF: low halves, OF: high halves), about 1.7x the u128 code's rate.  Five
  // accumulator registers rotate: iteration i adds a b_i into L0..L4, then
  // m p with m = L0 (-p^-1) zeroes L0, which becomes the next top limb.
  // Bounds (p < 2^255): t + a b_i + m p < 2^320, so no carry leaves L4.
  static inline T mul_adx(const T& a, const T& b) {
    alignas(64) static const uint64_t PN[5] = {P[0], P[1], P[2], P[3], NINV};
    uint64_t r0 = 0, r1 = 0, r2 = 0, r3 = 0, r4 = 0, lo, hi;
#define ZKL_MONT_ITER(OFF, L0, L1, L2, L3, L4)                      \
  "movq " #OFF "(%[b]), %%rdx\n\t"                                 \
  "xorl %%eax, %%eax\n\t"                                          \
  "mulxq 0(%[a]), %[lo], %[hi]\n\t"                                \
  "adcxq %[lo], %[" #L0 "]\n\t"                                    \
  "adoxq %[hi], %[" #L1 "]\n\t"                                    \
  "mulxq 8(%[a]), %[lo], %[hi]\n\t"                                \
  "adcxq %[lo], %[" #L1 "]\n\t"                                    \
  "adoxq %[hi], %[" #L2 "]\n\t"                                    \
  "mulxq 16(%[a]), %[lo], %[hi]\n\t"                               \
  "adcxq %[lo], %[" #L2 "]\n\t"                                    \
  "adoxq %[hi], %[" #L3 "]\n\t"                                    \
  "mulxq 24(%[a]), %[lo], %[hi]\n\t"                               \
  "adcxq %[lo], %[" #L3 "]\n\t"                                    \
  "adoxq %[hi], %[" #L4 "]\n\t"                                    \
  "adcxq %%rax, %[" #L4 "]\n\t"                                    \
  "movq %[" #L0 "], %%rdx\n\t"                                     \
  "imulq 32(%[p]), %%rdx\n\t"                                      \
  "xorl %%eax, %%eax\n\t"                                          \
  "mulxq 0(%[p]), %[lo], %[hi]\n\t"                                \
  "adcxq %[lo], %[" #L0 "]\n\t"                                    \
  "adoxq %[hi], %[" #L1 "]\n\t"                                    \
  "mulxq 8(%[p]), %[lo], %[hi]\n\t"                                \
  "adcxq %[lo], %[" #L1 "]\n\t"                                    \
  "adoxq %[hi], %[" #L2 "]\n\t"                                    \
  "mulxq 16(%[p]), %[lo], %[hi]\n\t"                               \
  "adcxq %[lo], %[" #L2 "]\n\t"                                    \
  "adoxq %[hi], %[" #L3 "]\n\t"                                    \
  "mulxq 24(%[p]), %[lo], %[hi]\n\t"                               \
  "adcxq %[lo], %[" #L3 "]\n\t"                                    \
  "adoxq %[hi], %[" #L4 "]\n\t"                                    \
  "adcxq %%rax, %[" #L4 "]\n\t"
    asm(ZKL_MONT_ITER(0, r0, r1, r2, r3, r4)
        ZKL_MONT_ITER(8, r1, r2, r3, r4, r0)
        ZKL_MONT_ITER(16, r2, r3, r4, r0, r1)
        ZKL_MONT_ITER(24, r3, r4, r0, r1, r2)
        : [r0] "+&r"(r0), [r1] "+&r"(r1), [r2] "+&r"(r2), [r3] "+&r"(r3), [r4] "+&r"(r4),
          [lo] "=&r"(lo), [hi] "=&r"(hi)
        : [a] "r"(&a), [b] "r"(&b), [p] "r"(PN)
        : "rax", "rdx", "cc", "memory");
#undef ZKL_MONT_ITER
    uint64_t r[4] = {r4, r0, r1, r2};  // t < 2p < 2^256: r3 is zero
    if (geq_p(r)) sub_p(r);
    return st(r);
  }
#endif
  static inline T mul_portable(const T& a, const T& b) {
    uint64_t x[4], y[4], t[6] = {0, 0, 0, 0, 0, 0};
    ld(a, x);
    ld(b, y);
    for (int i = 0; i < 4; i++) {
      u128 c = 0;
      for (int j = 0; j < 4; j++) {
        c += (u128)x[j] * y[i] + t[j];
        t[j] = (uint64_t)c;
        c >>= 64;
      }
      c += t[4];
      t[4] = (uint64_t)c;
      t[5] = (uint64_t)(c >> 64);
      const uint64_t m = t[0] * NINV;
      c = ((u128)m * P[0] + t[0]) >> 64;
      for (int j = 1; j < 4; j++) {
        c += (u128)m * P[j] + t[j];
        t[j - 1] = (uint64_t)c;
        c >>= 64;
      }
      c += t[4];
      t[3] = (uint64_t)c;
      t[4] = t[5] + (uint64_t)(c >> 64);
    }
    uint64_t r[4] = {t[0], t[1], t[2], t[3]};
    if (t[4] || geq_p(r)) sub_p(r);
    return st(r);
  }
  static inline T zero() { return Fr255::zero(); }
  static inline T one() { return Fr255::one(); }  // Montgomery 1
  static inline T to_mont(const T& canon) {
    uint64_t r2[4] = {R2[0], R2[1], R2[2], R2[3]};
    return mul(canon, st(r2));
  }
  static inline T from_mont(const T& a) {
    T one_c = Fr255::zero();
    one_c.v[0] = 1;
    return mul(a, one_c);
  }
  static inline bool is_zero(const T& a) { return Fr255::is_zero(a); }
};

struct M61h {
  using T = uint64_t;
  static inline T add(T a, T b) { return M61::add(a, b); }
  static inline T sub(T a, T b) { return M61::sub(a, b); }
  static inline T mul(T a, T b) { return M61::mul(a, b); }
  static inline T zero() { return 0; }
  static inline T one() { return 1; }
  static inline T to_mont(T a) { return a; }
  static inline T from_mont(T a) { return a; }
  static inline bool is_zero(T a) { return a == 0; }
};

template <class F>
struct For;
template <>
struct For<Fr255> {
  using H = Fr;
};
template <>
struct For<M61> {
  using H = M61h;
};

// canonical little-endian bytes <-> storage form (Montgomery for Fr)
template <class F>
inline typename F::T from_canon(const uint8_t* b) {
  typename F::T r;
  memcpy(&r, b, F::kBytes);
  return For<F>::H::to_mont(r);
}
template <class F>
inline void to_canon(uint8_t* b, const typename F::T& x) {
  typename F::T c = For<F>::H::from_mont(x);
  memcpy(b, &c, F::kBytes);
}
// canonical value (not Montgomery) of a storage-form element
template <class F>
inline typename F::T canon_of(const typename F::T& x) {
  return For<F>::H::from_mont(x);
}
// x^e by square-and-multiply (storage form)
template <class F>
inline typename F::T pow(typename F::T x, const uint8_t* e_le, int nbytes) {
  using H = typename For<F>::H;
  typename F::T r = H::one();
  for (int i = nbytes * 8 - 1; i >= 0; i--) {
    r = H::mul(r, r);
    if ((e_le[i >> 3] >> (i & 7)) & 1) r = H::mul(r, x);
  }
  return r;
}

}  // namespace host
}  // namespace zkl
