// Prime-field arithmetic for the zkLoRA sumcheck path on sm_100a.
//
// Two fields, one interface (reference: pkg/src/zklora/field.py:9-12):
//   Fr255 : BLS12-381 scalar field, 8 x 32-bit limbs, Montgomery form with
//           R = 2^256; device multiply is CIOS with 64-bit IMAD.WIDE limb
//           products and add-with-carry chains.
//   M61   : 2^61 - 1 (the reference's test field), canonical u64 form.
//
// Device storage is array-of-structs: one element = 32 B (Fr255) or 8 B
// (M61), limbs little-endian, so a canonical element's bytes equal the
// reference's 32-byte little-endian encoding (field.py:58-60).
#pragma once
#include <stdint.h>

// Montgomery multiplies keep their outer CIOS loop ROLLED by default: the
// round kernels are latency-bound single passes, and a fully unrolled
// multiply (~500 SASS instructions) re-fetched from L2 every round costs more
// than the loop overhead.  -DZKL_MUL_UNROLLED restores full unrolling (the
// throughput-bound kernels may prefer it).
#if defined(ZKL_MUL_UNROLLED)
#define ZKL_CIOS_LOOP _Pragma("unroll")
#else
#define ZKL_CIOS_LOOP _Pragma("unroll 1")
#endif

#if defined(__CUDACC__)
#define ZKL_HD __host__ __device__ __forceinline__
#define ZKL_D __device__ __forceinline__
#else
#define ZKL_HD inline
#define ZKL_D inline
#endif

namespace zkl {

// ---------------------------------------------------------------------------
// Fr255
struct alignas(16) fr_t {
  uint32_t v[8];
};

struct Fr255 {
  using T = fr_t;
  static constexpr int kBytes = 32;
  static constexpr int kId = 0;
  // p = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
  static constexpr uint32_t P0 = 0x00000001u, P1 = 0xFFFFFFFFu, P2 = 0xFFFE5BFEu,
                            P3 = 0x53BDA402u, P4 = 0x09A1D805u, P5 = 0x3339D808u,
                            P6 = 0x299D7D48u, P7 = 0x73EDA753u;
  // R mod p (Montgomery one) and R^2 mod p, R = 2^256
  ZKL_HD static T zero() { T r; for (int i = 0; i < 8; i++) r.v[i] = 0; return r; }
  ZKL_HD static T one() {
    T r; r.v[0] = 0xfffffffeu; r.v[1] = 0x00000001u; r.v[2] = 0x00034802u;
    r.v[3] = 0x5884b7fau; r.v[4] = 0xecbc4ff5u; r.v[5] = 0x998c4fefu;
    r.v[6] = 0xacc5056fu; r.v[7] = 0x1824b159u; return r;
  }
  ZKL_HD static T r2() {
    T r; r.v[0] = 0xf3f29c6du; r.v[1] = 0xc999e990u; r.v[2] = 0x87925c23u;
    r.v[3] = 0x2b6cedcbu; r.v[4] = 0x7254398fu; r.v[5] = 0x05d31496u;
    r.v[6] = 0x9f59ff11u; r.v[7] = 0x0748d9d9u; return r;
  }
  ZKL_HD static T modulus() {
    T r; r.v[0] = P0; r.v[1] = P1; r.v[2] = P2; r.v[3] = P3;
    r.v[4] = P4; r.v[5] = P5; r.v[6] = P6; r.v[7] = P7; return r;
  }

  ZKL_HD static bool is_zero(const T& a) {
    uint32_t x = 0;
    for (int i = 0; i < 8; i++) x |= a.v[i];
    return x == 0;
  }
  ZKL_HD static bool eq(const T& a, const T& b) {
    uint32_t x = 0;
    for (int i = 0; i < 8; i++) x |= a.v[i] ^ b.v[i];
    return x == 0;
  }

  // -------- portable (host + device) reference implementations ----------
  ZKL_HD static bool geq_p_portable(const T& a) {
    const T p = modulus();
    for (int i = 7; i >= 0; i--) {
      if (a.v[i] > p.v[i]) return true;
      if (a.v[i] < p.v[i]) return false;
    }
    return true;
  }
  ZKL_HD static T sub_p_portable(const T& a) {
    const T p = modulus();
    T r; int64_t br = 0;
    for (int i = 0; i < 8; i++) {
      int64_t d = (int64_t)a.v[i] - (int64_t)p.v[i] + br;
      r.v[i] = (uint32_t)d; br = d >> 32;
    }
    return r;
  }
  ZKL_HD static T add_portable(const T& a, const T& b) {
    T r; uint64_t c = 0;
    for (int i = 0; i < 8; i++) {
      uint64_t s = (uint64_t)a.v[i] + b.v[i] + c;
      r.v[i] = (uint32_t)s; c = s >> 32;
    }
    // a + b < 2p < 2^256: no carry out
    if (geq_p_portable(r)) r = sub_p_portable(r);
    return r;
  }
  ZKL_HD static T sub_portable(const T& a, const T& b) {
    T r; int64_t br = 0;
    for (int i = 0; i < 8; i++) {
      int64_t d = (int64_t)a.v[i] - (int64_t)b.v[i] + br;
      r.v[i] = (uint32_t)d; br = d >> 32;
    }
    if (br) {  // add p back
      const T p = modulus(); uint64_t c = 0;
      for (int i = 0; i < 8; i++) {
        uint64_t s = (uint64_t)r.v[i] + p.v[i] + c;
        r.v[i] = (uint32_t)s; c = s >> 32;
      }
    }
    return r;
  }
  // CIOS Montgomery multiply, 32-bit limbs, n' = -p^-1 mod 2^32 = 0xffffffff.
  ZKL_HD static T mul_portable(const T& a, const T& b) {
    const T p = modulus();
    uint32_t t[10] = {0};
    for (int i = 0; i < 8; i++) {
      uint64_t c = 0;
      for (int j = 0; j < 8; j++) {
        uint64_t s = (uint64_t)a.v[j] * b.v[i] + t[j] + c;
        t[j] = (uint32_t)s; c = s >> 32;
      }
      uint64_t s = (uint64_t)t[8] + c; t[8] = (uint32_t)s; t[9] = (uint32_t)(s >> 32);
      uint32_t m = t[0] * 0xffffffffu;
      c = ((uint64_t)m * p.v[0] + t[0]) >> 32;
      for (int j = 1; j < 8; j++) {
        uint64_t s2 = (uint64_t)m * p.v[j] + t[j] + c;
        t[j - 1] = (uint32_t)s2; c = s2 >> 32;
      }
      s = (uint64_t)t[8] + c; t[7] = (uint32_t)s;
      t[8] = t[9] + (uint32_t)(s >> 32);
    }
    T r; for (int i = 0; i < 8; i++) r.v[i] = t[i];
    if (t[8] || geq_p_portable(r)) r = sub_p_portable(r);
    return r;
  }

#if defined(__CUDA_ARCH__)
  // -------- device fast paths (PTX carry chains) ----------
  ZKL_D static T reduce_once(const T& a) {  // a < 2p -> a mod p
    T r; uint32_t br;
    asm("sub.cc.u32  %0, %9, %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;\n\t"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]),
          "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7]), "=r"(br)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
          "r"(a.v[6]), "r"(a.v[7]), "n"(P0), "n"(P1), "n"(P2), "n"(P3), "n"(P4), "n"(P5),
          "n"(P6), "n"(P7));
    // borrow (br = 0xffffffff) -> a < p, keep a
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = br ? a.v[i] : r.v[i];
    return r;
  }
  ZKL_D static T add(const T& a, const T& b) {
    T s;
    asm("add.cc.u32  %0, %8, %16;\n\t"
        "addc.cc.u32 %1, %9, %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;\n\t"
        : "=r"(s.v[0]), "=r"(s.v[1]), "=r"(s.v[2]), "=r"(s.v[3]), "=r"(s.v[4]),
          "=r"(s.v[5]), "=r"(s.v[6]), "=r"(s.v[7])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
          "r"(a.v[6]), "r"(a.v[7]), "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]),
          "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    return reduce_once(s);
  }
  ZKL_D static T sub(const T& a, const T& b) {
    T d; uint32_t br;
    asm("sub.cc.u32  %0, %9, %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;\n\t"
        : "=r"(d.v[0]), "=r"(d.v[1]), "=r"(d.v[2]), "=r"(d.v[3]), "=r"(d.v[4]),
          "=r"(d.v[5]), "=r"(d.v[6]), "=r"(d.v[7]), "=r"(br)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
          "r"(a.v[6]), "r"(a.v[7]), "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]),
          "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    // on borrow add p (br is 0 or 0xffffffff: mask p)
    T r;
    asm("add.cc.u32  %0, %8, %16;\n\t"
        "addc.cc.u32 %1, %9, %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;\n\t"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]),
          "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7])
        : "r"(d.v[0]), "r"(d.v[1]), "r"(d.v[2]), "r"(d.v[3]), "r"(d.v[4]), "r"(d.v[5]),
          "r"(d.v[6]), "r"(d.v[7]), "r"(br & P0), "r"(br & P1), "r"(br & P2), "r"(br & P3),
          "r"(br & P4), "r"(br & P5), "r"(br & P6), "r"(br & P7));
    return r;
  }

  // One CIOS outer step: t[0..8] += a * bi; then Montgomery-reduce one limb
  // and shift.  Invariant (a, b < p): t < 2p < 2^256 between steps.
  // Limb products are 64-bit IMAD.WIDE.U32 (full rate; a mad.lo/mad.hi pair
  // costs three times the IMAD-pipe slots): the even-limb products of a row
  // tile t without overlap, the odd ones likewise 32 bits up, so each row is
  // two add-with-carry chains.  tools/mont_bench.cu: 1.2-1.3x the products/s
  // of the mad.lo/hi.cc formulation.
  ZKL_D static void acc8(uint32_t& x0, uint32_t& x1, uint32_t& x2, uint32_t& x3, uint32_t& x4,
                         uint32_t& x5, uint32_t& x6, uint32_t& x7, uint32_t& x8, uint32_t w0,
                         uint32_t w1, uint32_t w2, uint32_t w3, uint32_t w4, uint32_t w5,
                         uint32_t w6, uint32_t w7) {
    asm("add.cc.u32 %0, %0, %9;\n\taddc.cc.u32 %1, %1, %10;\n\taddc.cc.u32 %2, %2, %11;\n\t"
        "addc.cc.u32 %3, %3, %12;\n\taddc.cc.u32 %4, %4, %13;\n\taddc.cc.u32 %5, %5, %14;\n\t"
        "addc.cc.u32 %6, %6, %15;\n\taddc.cc.u32 %7, %7, %16;\n\taddc.u32 %8, %8, 0;"
        : "+r"(x0), "+r"(x1), "+r"(x2), "+r"(x3), "+r"(x4), "+r"(x5), "+r"(x6), "+r"(x7),
          "+r"(x8)
        : "r"(w0), "r"(w1), "r"(w2), "r"(w3), "r"(w4), "r"(w5), "r"(w6), "r"(w7));
  }
  // x[0..7] += w[0..7], no carry out of the top word
  ZKL_D static void acc8n(uint32_t& x0, uint32_t& x1, uint32_t& x2, uint32_t& x3, uint32_t& x4,
                          uint32_t& x5, uint32_t& x6, uint32_t& x7, uint32_t w0, uint32_t w1,
                          uint32_t w2, uint32_t w3, uint32_t w4, uint32_t w5, uint32_t w6,
                          uint32_t w7) {
    asm("add.cc.u32 %0, %0, %8;\n\taddc.cc.u32 %1, %1, %9;\n\taddc.cc.u32 %2, %2, %10;\n\t"
        "addc.cc.u32 %3, %3, %11;\n\taddc.cc.u32 %4, %4, %12;\n\taddc.cc.u32 %5, %5, %13;\n\t"
        "addc.cc.u32 %6, %6, %14;\n\taddc.u32 %7, %7, %15;"
        : "+r"(x0), "+r"(x1), "+r"(x2), "+r"(x3), "+r"(x4), "+r"(x5), "+r"(x6), "+r"(x7)
        : "r"(w0), "r"(w1), "r"(w2), "r"(w3), "r"(w4), "r"(w5), "r"(w6), "r"(w7));
  }
  ZKL_D static void cios_step(uint32_t t[9], const T& a, uint32_t bi) {
#define ZKL_LO(x) ((uint32_t)(x))
#define ZKL_HI(x) ((uint32_t)((x) >> 32))
    const uint64_t e0 = (uint64_t)a.v[0] * bi, e2 = (uint64_t)a.v[2] * bi,
                   e4 = (uint64_t)a.v[4] * bi, e6 = (uint64_t)a.v[6] * bi;
    const uint64_t o1 = (uint64_t)a.v[1] * bi, o3 = (uint64_t)a.v[3] * bi,
                   o5 = (uint64_t)a.v[5] * bi, o7 = (uint64_t)a.v[7] * bi;
    acc8(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], ZKL_LO(e0), ZKL_HI(e0),
         ZKL_LO(e2), ZKL_HI(e2), ZKL_LO(e4), ZKL_HI(e4), ZKL_LO(e6), ZKL_HI(e6));
    acc8n(t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], ZKL_LO(o1), ZKL_HI(o1), ZKL_LO(o3),
          ZKL_HI(o3), ZKL_LO(o5), ZKL_HI(o5), ZKL_LO(o7), ZKL_HI(o7));
    // m = -t0 (n' = -1 mod 2^32 since p0 = 1); t += m p, whose low limb
    // zeroes t0 with carry (t0 != 0)
    const uint32_t m = 0u - t[0];
    const uint64_t f2 = (uint64_t)m * P2, f4 = (uint64_t)m * P4, f6 = (uint64_t)m * P6;
    const uint64_t g1 = (uint64_t)m * P1, g3 = (uint64_t)m * P3, g5 = (uint64_t)m * P5,
                   g7 = (uint64_t)m * P7;
    acc8(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], m, 0u, ZKL_LO(f2), ZKL_HI(f2),
         ZKL_LO(f4), ZKL_HI(f4), ZKL_LO(f6), ZKL_HI(f6));
    acc8n(t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], ZKL_LO(g1), ZKL_HI(g1), ZKL_LO(g3),
          ZKL_HI(g3), ZKL_LO(g5), ZKL_HI(g5), ZKL_LO(g7), ZKL_HI(g7));
#undef ZKL_LO
#undef ZKL_HI
    // shift right one limb (t0 is now zero)
#pragma unroll
    for (int j = 0; j < 8; j++) t[j] = t[j + 1];
    t[8] = 0;
  }
  // b <- b rotated by one limb (rolled CIOS loops consume b.v[0] each step,
  // so no limb is ever indexed dynamically)
  ZKL_D static void rot(T& b) {
    const uint32_t x = b.v[0];
#pragma unroll
    for (int k = 0; k < 7; k++) b.v[k] = b.v[k + 1];
    b.v[7] = x;
  }
  // by two limbs (the loops run two CIOS steps per iteration)
  ZKL_D static void rot2(T& b) {
    const uint32_t x = b.v[0], y = b.v[1];
#pragma unroll
    for (int k = 0; k < 6; k++) b.v[k] = b.v[k + 2];
    b.v[6] = x;
    b.v[7] = y;
  }
  ZKL_D static T mul_inl(const T& a, T b) {
    uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    ZKL_CIOS_LOOP
    for (int i = 0; i < 8; i += 2) {
      cios_step(t, a, b.v[0]);
      cios_step(t, a, b.v[1]);
      rot2(b);
    }
    T r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = t[i];
    return reduce_once(r);
  }
  // Compact form used everywhere: the outer CIOS loop stays rolled (the next
  // limb of b is rotated into place, so nothing is dynamically indexed).  A
  // fully unrolled multiply is ~300 SASS instructions (~5 KB); inlining that
  // at every call site overflows the instruction cache, which dominated the
  // latency-bound single-warp stretches of a round ("I-cache").
  // Arguments and results travel BY VALUE: with references the ABI spills
  // them (and any kernel-parameter struct they point into) to local memory.
  static __device__ __noinline__ T mul(T a, T b) { return mul_inl(a, b); }
  struct Pair {
    T x, y;
  };
  // two independent products with interleaved carry chains (ILP 2), one call
  static __device__ __noinline__ Pair mul2_call(T a, T b, T c, T d) {
    uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, u[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    ZKL_CIOS_LOOP
    for (int i = 0; i < 8; i += 2) {
      cios_step(t, a, b.v[0]);
      cios_step(u, c, d.v[0]);
      cios_step(t, a, b.v[1]);
      cios_step(u, c, d.v[1]);
      rot2(b);
      rot2(d);
    }
    Pair p;
#pragma unroll
    for (int i = 0; i < 8; i++) { p.x.v[i] = t[i]; p.y.v[i] = u[i]; }
    p.x = reduce_once(p.x);
    p.y = reduce_once(p.y);
    return p;
  }
  ZKL_D static void mul2(const T& a, const T& b, const T& c, const T& d, T& ab, T& cd) {
    Pair p = mul2_call(a, b, c, d);
    ab = p.x;
    cd = p.y;
  }
  // three / four independent products with interleaved carry chains: the
  // latency of one product for the price of one call (args stay in registers)
  struct Triple {
    T x, y, z;
  };
  static __device__ __noinline__ Triple mul3_call(T a0, T b0, T a1, T b1, T a2, T b2) {
    uint32_t t[9] = {0}, u[9] = {0}, w[9] = {0};
    ZKL_CIOS_LOOP
    for (int i = 0; i < 8; i += 2) {
      cios_step(t, a0, b0.v[0]);
      cios_step(u, a1, b1.v[0]);
      cios_step(w, a2, b2.v[0]);
      cios_step(t, a0, b0.v[1]);
      cios_step(u, a1, b1.v[1]);
      cios_step(w, a2, b2.v[1]);
      rot2(b0);
      rot2(b1);
      rot2(b2);
    }
    Triple q;
#pragma unroll
    for (int i = 0; i < 8; i++) { q.x.v[i] = t[i]; q.y.v[i] = u[i]; q.z.v[i] = w[i]; }
    q.x = reduce_once(q.x);
    q.y = reduce_once(q.y);
    q.z = reduce_once(q.z);
    return q;
  }
  struct Quad {
    T x, y, z, w;
  };
  // r * a0, r * a1, r * a2, r * a3 (the fold of two tables' lo/hi halves)
  static __device__ __noinline__ Quad mul4r_call(T r, T a0, T a1, T a2, T a3) {
    uint32_t t[9] = {0}, u[9] = {0}, v[9] = {0}, w[9] = {0};
    ZKL_CIOS_LOOP
    for (int i = 0; i < 8; i += 2) {
      cios_step(t, a0, r.v[0]);
      cios_step(u, a1, r.v[0]);
      cios_step(v, a2, r.v[0]);
      cios_step(w, a3, r.v[0]);
      cios_step(t, a0, r.v[1]);
      cios_step(u, a1, r.v[1]);
      cios_step(v, a2, r.v[1]);
      cios_step(w, a3, r.v[1]);
      rot2(r);
    }
    Quad q;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      q.x.v[i] = t[i]; q.y.v[i] = u[i]; q.z.v[i] = v[i]; q.w.v[i] = w[i];
    }
    q.x = reduce_once(q.x);
    q.y = reduce_once(q.y);
    q.z = reduce_once(q.z);
    q.w = reduce_once(q.w);
    return q;
  }
  static __device__ __noinline__ Quad mul4_call(T a0, T b0, T a1, T b1, T a2, T b2, T a3, T b3) {
    uint32_t t[9] = {0}, u[9] = {0}, v[9] = {0}, w[9] = {0};
    ZKL_CIOS_LOOP
    for (int i = 0; i < 8; i += 2) {
      cios_step(t, a0, b0.v[0]);
      cios_step(u, a1, b1.v[0]);
      cios_step(v, a2, b2.v[0]);
      cios_step(w, a3, b3.v[0]);
      cios_step(t, a0, b0.v[1]);
      cios_step(u, a1, b1.v[1]);
      cios_step(v, a2, b2.v[1]);
      cios_step(w, a3, b3.v[1]);
      rot2(b0);
      rot2(b1);
      rot2(b2);
      rot2(b3);
    }
    Quad q;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      q.x.v[i] = t[i]; q.y.v[i] = u[i]; q.z.v[i] = v[i]; q.w.v[i] = w[i];
    }
    q.x = reduce_once(q.x);
    q.y = reduce_once(q.y);
    q.z = reduce_once(q.z);
    q.w = reduce_once(q.w);
    return q;
  }
  ZKL_D static void mul3(const T& a0, const T& b0, const T& a1, const T& b1, const T& a2,
                         const T& b2, T& o0, T& o1, T& o2) {
    Triple q = mul3_call(a0, b0, a1, b1, a2, b2);
    o0 = q.x; o1 = q.y; o2 = q.z;
  }
  ZKL_D static void mul4(const T& a0, const T& b0, const T& a1, const T& b1, const T& a2,
                         const T& b2, const T& a3, const T& b3, T& o0, T& o1, T& o2, T& o3) {
    Quad q = mul4_call(a0, b0, a1, b1, a2, b2, a3, b3);
    o0 = q.x; o1 = q.y; o2 = q.z; o3 = q.w;
  }
  ZKL_D static void mul4r(const T& r, T& a0, T& a1, T& a2, T& a3) {
    Quad q = mul4r_call(r, a0, a1, a2, a3);
    a0 = q.x; a1 = q.y; a2 = q.z; a3 = q.w;
  }
#else
  static T reduce_once(const T& a) { return geq_p_portable(a) ? sub_p_portable(a) : a; }
  static T add(const T& a, const T& b) { return add_portable(a, b); }
  static T sub(const T& a, const T& b) { return sub_portable(a, b); }
  static T mul(const T& a, const T& b) { return mul_portable(a, b); }
  static T mul_inl(const T& a, const T& b) { return mul_portable(a, b); }
  static void mul2(const T& a, const T& b, const T& c, const T& d, T& ab, T& cd) {
    ab = mul_portable(a, b);
    cd = mul_portable(c, d);
  }
  static void mul3(const T& a0, const T& b0, const T& a1, const T& b1, const T& a2, const T& b2,
                   T& o0, T& o1, T& o2) {
    o0 = mul_portable(a0, b0); o1 = mul_portable(a1, b1); o2 = mul_portable(a2, b2);
  }
  static void mul4(const T& a0, const T& b0, const T& a1, const T& b1, const T& a2, const T& b2,
                   const T& a3, const T& b3, T& o0, T& o1, T& o2, T& o3) {
    o0 = mul_portable(a0, b0); o1 = mul_portable(a1, b1);
    o2 = mul_portable(a2, b2); o3 = mul_portable(a3, b3);
  }
  static void mul4r(const T& r, T& a0, T& a1, T& a2, T& a3) {
    a0 = mul_portable(r, a0); a1 = mul_portable(r, a1);
    a2 = mul_portable(r, a2); a3 = mul_portable(r, a3);
  }
#endif

  ZKL_HD static T neg(const T& a) { return sub(zero(), a); }
  ZKL_HD static T to_mont(const T& a) { return mul(a, r2()); }  // a < p
  ZKL_HD static T from_mont(const T& a) {
    T one_c = zero(); one_c.v[0] = 1;
    return mul(a, one_c);
  }
  // Montgomery form of a signed 64-bit integer (negatives as p - |x|).
  ZKL_HD static T from_i64(int64_t x) {
    uint64_t m = x < 0 ? (uint64_t)(-(x + 1)) + 1u : (uint64_t)x;
    T a = zero(); a.v[0] = (uint32_t)m; a.v[1] = (uint32_t)(m >> 32);
    T r = mul(a, r2());
    return x < 0 ? neg(r) : r;
  }
  ZKL_HD static T from_u32(uint32_t x) {
    T a = zero(); a.v[0] = x;
    return mul(a, r2());
  }
};

// ---------------------------------------------------------------------------
// Mersenne-61
struct M61 {
  using T = uint64_t;
  static constexpr int kBytes = 8;
  static constexpr int kId = 1;
  static constexpr uint64_t P = (1ull << 61) - 1;
  ZKL_HD static T zero() { return 0; }
  ZKL_HD static T one() { return 1; }
  ZKL_HD static T modulus() { return P; }
  ZKL_HD static bool is_zero(T a) { return a == 0; }
  ZKL_HD static bool eq(T a, T b) { return a == b; }
  ZKL_HD static T add(T a, T b) { T s = a + b; return s >= P ? s - P : s; }
  ZKL_HD static T sub(T a, T b) { return a >= b ? a - b : a + P - b; }
  ZKL_HD static T neg(T a) { return a ? P - a : 0; }
  ZKL_HD static T mul(T a, T b) {
#if defined(__CUDA_ARCH__)
    uint64_t lo = a * b, hi = __umul64hi(a, b);
#else
    unsigned __int128 w = (unsigned __int128)a * b;
    uint64_t lo = (uint64_t)w, hi = (uint64_t)(w >> 64);
#endif
    uint64_t r = (lo & P) + ((lo >> 61) | (hi << 3));
    r = (r & P) + (r >> 61);
    return r >= P ? r - P : r;
  }
  ZKL_HD static void mul2(T a, T b, T c, T d, T& ab, T& cd) {
    ab = mul(a, b);
    cd = mul(c, d);
  }
  ZKL_HD static void mul3(T a0, T b0, T a1, T b1, T a2, T b2, T& o0, T& o1, T& o2) {
    o0 = mul(a0, b0); o1 = mul(a1, b1); o2 = mul(a2, b2);
  }
  ZKL_HD static void mul4(T a0, T b0, T a1, T b1, T a2, T b2, T a3, T b3, T& o0, T& o1, T& o2,
                          T& o3) {
    o0 = mul(a0, b0); o1 = mul(a1, b1); o2 = mul(a2, b2); o3 = mul(a3, b3);
  }
  ZKL_HD static void mul4r(T r, T& a0, T& a1, T& a2, T& a3) {
    a0 = mul(r, a0); a1 = mul(r, a1); a2 = mul(r, a2); a3 = mul(r, a3);
  }
  ZKL_HD static T to_mont(T a) { return a; }
  ZKL_HD static T from_mont(T a) { return a; }
  ZKL_HD static T from_i64(int64_t x) {
    uint64_t m = x < 0 ? (uint64_t)(-(x + 1)) + 1u : (uint64_t)x;
    m = (m & P) + (m >> 61);
    if (m >= P) m -= P;
    return x < 0 ? neg(m) : m;
  }
  ZKL_HD static T from_u32(uint32_t x) { return x; }
};

// ---------------------------------------------------------------------------
// canonical little-endian bytes <-> field (host side, scalars)
template <class F>
inline typename F::T load_canon(const uint8_t* b) {
  typename F::T r;
  const uint8_t* s = b;
  uint8_t* d = reinterpret_cast<uint8_t*>(&r);
  for (int i = 0; i < F::kBytes; i++) d[i] = s[i];
  return F::to_mont(r);
}
template <class F>
inline void store_canon(uint8_t* b, const typename F::T& x) {
  typename F::T c = F::from_mont(x);
  const uint8_t* s = reinterpret_cast<const uint8_t*>(&c);
  for (int i = 0; i < F::kBytes; i++) b[i] = s[i];
}

// Fermat inverse (host or device; slow on device, used on host for the one
// top-level inversion of a batch).
template <class F>
ZKL_HD typename F::T pow_p_minus_2(const typename F::T& a);

}  // namespace zkl
