// Integer-matrix x field-vector products for the factored zkMat prover.
//
// Reference context: the zkMat claim of gadgets.py:210-251 is proven without
// materialising its 2^(d0+d1+d2) replicated tables; instead every MLE partial
// evaluation it needs is a matrix-vector product against an eq-vector:
//   B E_v, C E_v, A (B E_v)   (row products,  y = M x)
//   E_rho_u^T A, E_rho_u^T C, E_rho_w^T B   (column products, y = M^T x)
// (derivation: DESIGN.md "Factored zkMat").
//
// Fr255 with integer matrices (int16 / int32 / int64): multiply-accumulate
// into a wide (320/384-bit) integer accumulator with one 16-IMAD row of
// mad.lo/hi.cc per 32-bit matrix word and no modular reduction in the inner
// loop.  Signed entries use offset binary: sum (s + o) x - o * sum x, so the
// inner loop is unsigned; the wide sum is reduced mod p once per output.
// Other combinations (M61, field-valued matrices) multiply-add in the field.
#include <cstdlib>

#include "ops.cuh"

namespace zkl {

// ---------------------------------------------------------------------------
// wide accumulator (Fr255)
template <int W>
struct Wide {
  uint32_t w[W];
};

// a[0..9] += u * x  (10-limb accumulator)
ZKL_D void mac10(Wide<10>& a, uint32_t u, const fr_t& x) {
  asm("mad.lo.cc.u32  %0, %10, %18, %0;\n\t"
      "madc.lo.cc.u32 %1, %11, %18, %1;\n\t"
      "madc.lo.cc.u32 %2, %12, %18, %2;\n\t"
      "madc.lo.cc.u32 %3, %13, %18, %3;\n\t"
      "madc.lo.cc.u32 %4, %14, %18, %4;\n\t"
      "madc.lo.cc.u32 %5, %15, %18, %5;\n\t"
      "madc.lo.cc.u32 %6, %16, %18, %6;\n\t"
      "madc.lo.cc.u32 %7, %17, %18, %7;\n\t"
      "addc.cc.u32    %8, %8, 0;\n\t"
      "addc.u32       %9, %9, 0;\n\t"
      "mad.hi.cc.u32  %1, %10, %18, %1;\n\t"
      "madc.hi.cc.u32 %2, %11, %18, %2;\n\t"
      "madc.hi.cc.u32 %3, %12, %18, %3;\n\t"
      "madc.hi.cc.u32 %4, %13, %18, %4;\n\t"
      "madc.hi.cc.u32 %5, %14, %18, %5;\n\t"
      "madc.hi.cc.u32 %6, %15, %18, %6;\n\t"
      "madc.hi.cc.u32 %7, %16, %18, %7;\n\t"
      "madc.hi.cc.u32 %8, %17, %18, %8;\n\t"
      "addc.u32       %9, %9, 0;\n\t"
      : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]), "+r"(a.w[5]),
        "+r"(a.w[6]), "+r"(a.w[7]), "+r"(a.w[8]), "+r"(a.w[9])
      : "r"(x.v[0]), "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]),
        "r"(x.v[6]), "r"(x.v[7]), "r"(u));
}

// a[off..off+9] += u * x for a 12-limb accumulator, off in {0, 1}
template <int OFF>
ZKL_D void mac12(Wide<12>& a, uint32_t u, const fr_t& x) {
  uint32_t* w = a.w + OFF;
  if (OFF == 0) {
    asm("mad.lo.cc.u32  %0, %12, %20, %0;\n\t"
        "madc.lo.cc.u32 %1, %13, %20, %1;\n\t"
        "madc.lo.cc.u32 %2, %14, %20, %2;\n\t"
        "madc.lo.cc.u32 %3, %15, %20, %3;\n\t"
        "madc.lo.cc.u32 %4, %16, %20, %4;\n\t"
        "madc.lo.cc.u32 %5, %17, %20, %5;\n\t"
        "madc.lo.cc.u32 %6, %18, %20, %6;\n\t"
        "madc.lo.cc.u32 %7, %19, %20, %7;\n\t"
        "addc.cc.u32    %8, %8, 0;\n\t"
        "addc.cc.u32    %9, %9, 0;\n\t"
        "addc.cc.u32    %10, %10, 0;\n\t"
        "addc.u32       %11, %11, 0;\n\t"
        "mad.hi.cc.u32  %1, %12, %20, %1;\n\t"
        "madc.hi.cc.u32 %2, %13, %20, %2;\n\t"
        "madc.hi.cc.u32 %3, %14, %20, %3;\n\t"
        "madc.hi.cc.u32 %4, %15, %20, %4;\n\t"
        "madc.hi.cc.u32 %5, %16, %20, %5;\n\t"
        "madc.hi.cc.u32 %6, %17, %20, %6;\n\t"
        "madc.hi.cc.u32 %7, %18, %20, %7;\n\t"
        "madc.hi.cc.u32 %8, %19, %20, %8;\n\t"
        "addc.cc.u32    %9, %9, 0;\n\t"
        "addc.cc.u32    %10, %10, 0;\n\t"
        "addc.u32       %11, %11, 0;\n\t"
        : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]),
          "+r"(w[7]), "+r"(w[8]), "+r"(w[9]), "+r"(w[10]), "+r"(w[11])
        : "r"(x.v[0]), "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]),
          "r"(x.v[6]), "r"(x.v[7]), "r"(u));
  } else {
    asm("mad.lo.cc.u32  %0, %11, %19, %0;\n\t"
        "madc.lo.cc.u32 %1, %12, %19, %1;\n\t"
        "madc.lo.cc.u32 %2, %13, %19, %2;\n\t"
        "madc.lo.cc.u32 %3, %14, %19, %3;\n\t"
        "madc.lo.cc.u32 %4, %15, %19, %4;\n\t"
        "madc.lo.cc.u32 %5, %16, %19, %5;\n\t"
        "madc.lo.cc.u32 %6, %17, %19, %6;\n\t"
        "madc.lo.cc.u32 %7, %18, %19, %7;\n\t"
        "addc.cc.u32    %8, %8, 0;\n\t"
        "addc.cc.u32    %9, %9, 0;\n\t"
        "addc.u32       %10, %10, 0;\n\t"
        "mad.hi.cc.u32  %1, %11, %19, %1;\n\t"
        "madc.hi.cc.u32 %2, %12, %19, %2;\n\t"
        "madc.hi.cc.u32 %3, %13, %19, %3;\n\t"
        "madc.hi.cc.u32 %4, %14, %19, %4;\n\t"
        "madc.hi.cc.u32 %5, %15, %19, %5;\n\t"
        "madc.hi.cc.u32 %6, %16, %19, %6;\n\t"
        "madc.hi.cc.u32 %7, %17, %19, %7;\n\t"
        "madc.hi.cc.u32 %8, %18, %19, %8;\n\t"
        "addc.cc.u32    %9, %9, 0;\n\t"
        "addc.u32       %10, %10, 0;\n\t"
        : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]),
          "+r"(w[7]), "+r"(w[8]), "+r"(w[9]), "+r"(w[10])
        : "r"(x.v[0]), "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]),
          "r"(x.v[6]), "r"(x.v[7]), "r"(u));
  }
}

// X = lo + hi 2^256 (hi < 2^128) -> X mod p in Montgomery form (X already
// carries the factor R through x, so plain reduction mod p is what we want).
template <int W>
ZKL_D fr_t reduce_wide(const Wide<W>& a) {
  fr_t lo, hi = Fr255::zero();
#pragma unroll
  for (int i = 0; i < 8; i++) lo.v[i] = a.w[i];
#pragma unroll
  for (int i = 8; i < W; i++) hi.v[i - 8] = a.w[i];
  lo = Fr255::reduce_once(Fr255::reduce_once(lo));  // lo < 2^256 < 3p
  hi = Fr255::mul(hi, Fr255::r2());                 // hi * 2^256 mod p
  return Fr255::add(lo, hi);
}

// ---------------------------------------------------------------------------
// accumulation policies.  Signed integer entries use sign-magnitude: the
// shared x chunk is staged twice, as x and p - x, and every entry s picks
// (|s|, s < 0 ? p - x : x), so the wide accumulator only ever adds.
template <class F, class MT>
struct Mac;

template <>
struct Mac<Fr255, int16_t> {
  using Acc = Wide<10>;
  static constexpr bool kSigned = true;
  ZKL_D static void init(Acc& a) {
#pragma unroll
    for (int i = 0; i < 10; i++) a.w[i] = 0;
  }
  ZKL_D static void mac(Acc& a, int16_t s, const fr_t* xp, const fr_t* xn) {
    const bool neg = s < 0;
    mac10(a, (uint32_t)(neg ? -(int32_t)s : (int32_t)s), neg ? *xn : *xp);
  }
  ZKL_D static fr_t done(const Acc& a) { return reduce_wide<10>(a); }
};
template <>
struct Mac<Fr255, int32_t> {
  using Acc = Wide<10>;
  static constexpr bool kSigned = true;
  ZKL_D static void init(Acc& a) {
#pragma unroll
    for (int i = 0; i < 10; i++) a.w[i] = 0;
  }
  ZKL_D static void mac(Acc& a, int32_t s, const fr_t* xp, const fr_t* xn) {
    const bool neg = s < 0;
    mac10(a, neg ? (uint32_t)(-(int64_t)s) : (uint32_t)s, neg ? *xn : *xp);
  }
  ZKL_D static fr_t done(const Acc& a) { return reduce_wide<10>(a); }
};
template <>
struct Mac<Fr255, int64_t> {
  using Acc = Wide<12>;
  static constexpr bool kSigned = true;
  ZKL_D static void init(Acc& a) {
#pragma unroll
    for (int i = 0; i < 12; i++) a.w[i] = 0;
  }
  ZKL_D static void mac(Acc& a, int64_t s, const fr_t* xp, const fr_t* xn) {
    const bool neg = s < 0;
    const uint64_t u = neg ? (uint64_t)(-(s + 1)) + 1u : (uint64_t)s;
    const fr_t& x = neg ? *xn : *xp;
    mac12<0>(a, (uint32_t)u, x);
    if (u >> 32) mac12<1>(a, (uint32_t)(u >> 32), x);
  }
  ZKL_D static fr_t done(const Acc& a) { return reduce_wide<12>(a); }
};
template <class F, class MT>
struct Mac {  // generic: field arithmetic per entry (M61 ints, field-valued matrices)
  using T = typename F::T;
  using Acc = T;
  static constexpr bool kSigned = false;
  ZKL_D static void init(Acc& a) { a = F::zero(); }
  template <class V>
  ZKL_D static T lift(const V& s) { return F::from_i64((int64_t)s); }
  ZKL_D static T lift(const T& s) { return s; }
  ZKL_D static void mac(Acc& a, const MT& s, const T* xp, const T*) {
    a = F::add(a, F::mul(lift(s), *xp));
  }
  ZKL_D static T done(const Acc& a) { return a; }
};

// vector loads of VEC consecutive entries (16-byte aligned)
template <class MT, int VEC>
ZKL_D void load_vec(const MT* p, MT (&v)[VEC]) {
  static_assert((sizeof(MT) * VEC) % 16 == 0, "vector width");
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint4* d = reinterpret_cast<uint4*>(v);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(MT) * VEC / 16); i++) d[i] = __ldcs(q + i);
}

// stage x[lo, hi) (and p - x for signed entries) into shared memory
template <class F, bool SIGNED>
ZKL_D void stage_x(const typename F::T* x, uint64_t lo, uint64_t hi, typename F::T* xp,
                   typename F::T* xn) {
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const typename F::T v = x[i];
    xp[i - lo] = v;
    if (SIGNED) xn[i - lo] = F::neg(v);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// row products: part[chunk][r] = sum_{c in chunk} M[r, c] x[c]; thread per row,
// VEC entries of the row per vector load, x broadcast from shared memory.
template <class F, class MT, int VEC>
__global__ void __launch_bounds__(256)
    k_mv_rows(const MT* M, uint64_t rows, uint64_t cols, const typename F::T* x, uint64_t cch,
              typename F::T* part) {
  using T = typename F::T;
  using P = Mac<F, MT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* xp = reinterpret_cast<T*>(smem_raw);
  T* xn = xp + cch;
  const uint64_t c0 = blockIdx.y * cch;
  const uint64_t c1 = c0 + cch < cols ? c0 + cch : cols;
  stage_x<F, P::kSigned>(x, c0, c1, xp, xn);
  const uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  typename P::Acc acc;
  P::init(acc);
  const MT* row = M + r * cols;
  uint64_t c = c0;
  // U vector loads issued before their multiply-adds: a thread per row walks
  // its own row, so memory-level parallelism comes from loads in flight per
  // thread (ncu: long-scoreboard stalls dominated the one-load-at-a-time loop)
  constexpr int U = VEC == 1 ? 8 : 4;
  for (; c + U * VEC <= c1; c += U * VEC) {
    MT v[U][VEC];
#pragma unroll
    for (int u = 0; u < U; u++) {
      if constexpr (VEC == 1)
        v[u][0] = row[c + u];
      else
        load_vec<MT, VEC>(row + c + u * VEC, v[u]);
    }
#pragma unroll
    for (int u = 0; u < U; u++)
#pragma unroll
      for (int k = 0; k < VEC; k++)
        P::mac(acc, v[u][k], xp + (c - c0) + u * VEC + k, xn + (c - c0) + u * VEC + k);
  }
  for (; c + VEC <= c1; c += VEC) {
    MT v[VEC];
    if constexpr (VEC == 1)
      v[0] = row[c];
    else
      load_vec<MT, VEC>(row + c, v);
#pragma unroll
    for (int k = 0; k < VEC; k++) P::mac(acc, v[k], xp + (c - c0) + k, xn + (c - c0) + k);
  }
  for (; c < c1; c++) P::mac(acc, row[c], xp + (c - c0), xn + (c - c0));
  part[blockIdx.y * rows + r] = P::done(acc);
}

// column products: part[chunk][c] = sum_{r in chunk} x[r] M[r, c]; threads
// over columns (coalesced rows of M), x[r] broadcast from shared memory; for
// narrow matrices several row groups share a block and reduce in shared memory.
template <class F, class MT>
__global__ void __launch_bounds__(256)
    k_mv_cols(const MT* M, uint64_t rows, uint64_t cols, const typename F::T* x, int cw,
              uint64_t rch, typename F::T* part) {
  using T = typename F::T;
  using P = Mac<F, MT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* xp = reinterpret_cast<T*>(smem_raw);
  T* xn = xp + rch;                               // only staged for signed entries
  T* red = xp + (P::kSigned ? 2 : 1) * rch;       // 256 entries
  const uint64_t r0 = blockIdx.y * rch;
  const uint64_t r1 = r0 + rch < rows ? r0 + rch : rows;
  stage_x<F, P::kSigned>(x, r0, r1, xp, xn);
  const int tc = threadIdx.x % cw, rg = threadIdx.x / cw, ngrp = blockDim.x / cw;
  const uint64_t c = blockIdx.x * (uint64_t)cw + tc;
  typename P::Acc acc;
  P::init(acc);
  if (c < cols) {
    // four rows' loads in flight before their multiply-adds (see k_mv_rows)
    uint64_t r = r0 + rg;
    for (; r + 3 * ngrp < r1; r += 4 * ngrp) {
      MT v[4];
#pragma unroll
      for (int u = 0; u < 4; u++) v[u] = M[(r + u * ngrp) * cols + c];
#pragma unroll
      for (int u = 0; u < 4; u++)
        P::mac(acc, v[u], xp + (r + u * ngrp - r0), xn + (r + u * ngrp - r0));
    }
    for (; r < r1; r += ngrp) P::mac(acc, M[r * cols + c], xp + (r - r0), xn + (r - r0));
  }
  if (ngrp == 1) {
    if (c < cols) part[blockIdx.y * cols + c] = P::done(acc);
    return;
  }
  red[threadIdx.x] = P::done(acc);
  __syncthreads();
  if (rg == 0 && c < cols) {
    T v = red[tc];
    for (int g = 1; g < ngrp; g++) v = F::add(v, red[g * cw + tc]);
    part[blockIdx.y * cols + c] = v;
  }
}

// y[i] = sum_b part[b][i]; one warp per output
template <class F>
__global__ void __launch_bounds__(256)
    k_mv_reduce(const typename F::T* part, uint64_t nchunks, uint64_t n, typename F::T* y) {
  using T = typename F::T;
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = w; i < n; i += nw) {
    T v = F::zero();
    for (uint64_t b = lane; b < nchunks; b += 32) v = F::add(v, part[b * n + i]);
    v = warp_sum<F>(v);
    if (lane == 0) y[i] = v;
  }
}

// ===========================================================================
// Fast path (Fr255 x int16 / int64): per-limb 64-bit accumulators fed by
// mad.wide.u32 -- no carry chains in the inner loop.
//
// x (Montgomery form, 8 x 32-bit limbs x_l) is shared by all outputs.  Every
// signed entry s is made unsigned by offset binary, u = s + OFF, so
//   sum_c s_c x_c = sum_c u_c x_c - OFF * sum_c x_c,
// where OFF * sum x is ONE per-chunk constant K (x is shared).  Limb products
// u_k x_l (u_k < 2^16, x_l < 2^32) are accumulated in u64 without carries:
//   int16 (1 chunk):  e[l]   += u x_l                      (weight 2^(32 l))
//   int64 (4 chunks of 16 bits, u = s + 2^63):
//                     e[l]   += u0 x_l,  e[l+1] += u2 x_l  (weight 2^(32 l))
//                     o[l]   += u1 x_l,  o[l+1] += u3 x_l  (weight 2^(32 l + 16))
// Each accumulator takes < 2^49 per entry, so chunks of <= 2^15 entries
// never overflow.  The epilogue folds the accumulators into a wide integer,
// reduces it mod p once and subtracts K.  Cost per int16 entry: 8 mad.wide
// (vs ~20 carry-chained mad.lo/hi.cc in the wide-accumulator kernels above).
template <int CH>
struct LimbAcc {
  static constexpr int NE = CH == 1 ? 8 : 9;
  uint64_t e[NE];
  uint64_t o[CH == 1 ? 1 : 9];
  ZKL_D void zero() {
#pragma unroll
    for (int i = 0; i < NE; i++) e[i] = 0;
#pragma unroll
    for (int i = 0; i < (CH == 1 ? 1 : 9); i++) o[i] = 0;
  }
};

ZKL_D uint64_t madw(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
  return r;
}

ZKL_D void mac_u16(LimbAcc<1>& a, uint32_t u, const fr_t& x) {
#pragma unroll
  for (int l = 0; l < 8; l++) a.e[l] = madw(u, x.v[l], a.e[l]);
}
ZKL_D void mac_u64(LimbAcc<4>& a, uint64_t u, const fr_t& x) {
  const uint32_t u0 = (uint32_t)u & 0xffffu, u1 = (uint32_t)(u >> 16) & 0xffffu;
  const uint32_t u2 = (uint32_t)(u >> 32) & 0xffffu, u3 = (uint32_t)(u >> 48);
#pragma unroll
  for (int l = 0; l < 8; l++) {
    a.e[l] = madw(u0, x.v[l], a.e[l]);
    a.e[l + 1] = madw(u2, x.v[l], a.e[l + 1]);
    a.o[l] = madw(u1, x.v[l], a.o[l]);
    a.o[l + 1] = madw(u3, x.v[l], a.o[l + 1]);
  }
}

// wide integer sum_m e[m] 2^(32m) + o[m] 2^(32m+16) -> value mod p (storage)
template <int CH>
ZKL_D fr_t limb_reduce(const LimbAcc<CH>& a) {
  // 14 x 32-bit words are enough: max ~2^(64 + 32*8 + 16) < 2^448
  uint32_t w[14];
#pragma unroll
  for (int i = 0; i < 14; i++) w[i] = 0;
  uint64_t carry = 0;
  // even part: word i gets lo(e[i]) + hi(e[i-1]) + carry
#pragma unroll
  for (int i = 0; i < 14; i++) {
    uint64_t t = carry;
    if (i < LimbAcc<CH>::NE) t += (uint32_t)a.e[i];
    if (i >= 1 && i - 1 < LimbAcc<CH>::NE) t += a.e[i - 1] >> 32;
    w[i] = (uint32_t)t;
    carry = t >> 32;
  }
  if (CH != 1) {
    // odd part (offset 16 bits): add sum_m o[m] 2^(32m+16)
    uint64_t c2 = 0;
#pragma unroll
    for (int i = 0; i < 14; i++) {
      // bits of the odd sum landing in word i: lo16(o[i]) << 16 | bits from o[i-1] >> 16 ...
      uint64_t t = c2 + (uint64_t)w[i];
      if (i < 9) t += (uint64_t)((uint32_t)a.o[i] & 0xffffu) << 16;
      if (i >= 1 && i - 1 < 9) t += (a.o[i - 1] >> 16) & 0xffffffffull;
      if (i >= 2 && i - 2 < 9) t += a.o[i - 2] >> 48;
      w[i] = (uint32_t)t;
      c2 = t >> 32;
    }
  }
  fr_t lo, hi = Fr255::zero();
#pragma unroll
  for (int i = 0; i < 8; i++) lo.v[i] = w[i];
#pragma unroll
  for (int i = 8; i < 14; i++) hi.v[i - 8] = w[i];
  lo = Fr255::reduce_once(Fr255::reduce_once(lo));  // lo < 2^256 < 3p
  hi = Fr255::mul(hi, Fr255::r2());                 // hi < 2^192 < p: hi * 2^256 mod p
  return Fr255::add(lo, hi);
}

// raw accumulator words of one partial: int16 8 x u64, int64 18 x u64
template <int CH>
struct AccIO {
  static constexpr int NW = CH == 1 ? 8 : 18;
  ZKL_D static void store(uint64_t* dst, const LimbAcc<CH>& a) {
    uint4* d = reinterpret_cast<uint4*>(dst);
    if constexpr (CH == 1) {
#pragma unroll
      for (int i = 0; i < 4; i++) d[i] = make_uint4((uint32_t)a.e[2 * i], (uint32_t)(a.e[2 * i] >> 32),
                                                   (uint32_t)a.e[2 * i + 1],
                                                   (uint32_t)(a.e[2 * i + 1] >> 32));
    } else {
      uint64_t w[18];
#pragma unroll
      for (int i = 0; i < 9; i++) { w[i] = a.e[i]; w[9 + i] = a.o[i]; }
#pragma unroll
      for (int i = 0; i < 9; i++)
        d[i] = make_uint4((uint32_t)w[2 * i], (uint32_t)(w[2 * i] >> 32), (uint32_t)w[2 * i + 1],
                          (uint32_t)(w[2 * i + 1] >> 32));
    }
  }
  // red.global.add.u64 of the raw words into a zeroed accumulator record
  ZKL_D static void atomic_add(uint64_t* dst, const LimbAcc<CH>& a) {
    unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
    if constexpr (CH == 1) {
#pragma unroll
      for (int i = 0; i < 8; i++) atomicAdd(d + i, (unsigned long long)a.e[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 9; i++) {
        atomicAdd(d + i, (unsigned long long)a.e[i]);
        atomicAdd(d + 9 + i, (unsigned long long)a.o[i]);
      }
    }
  }
  ZKL_D static void add(LimbAcc<CH>& a, const uint64_t* src) {
    const uint4* q = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int i = 0; i < NW / 2; i++) {
      const uint4 v = q[i];
      const uint64_t w0 = ((uint64_t)v.y << 32) | v.x, w1 = ((uint64_t)v.w << 32) | v.z;
      if constexpr (CH == 1) {
        a.e[2 * i] += w0;
        a.e[2 * i + 1] += w1;
      } else {
        const int j0 = 2 * i, j1 = 2 * i + 1;
        if (j0 < 9) a.e[j0] += w0; else a.o[j0 - 9] += w0;
        if (j1 < 9) a.e[j1] += w1; else a.o[j1 - 9] += w1;
      }
    }
  }
};

template <class MT>
ZKL_D void mac_entry(LimbAcc<sizeof(MT) == 2 ? 1 : 4>& acc, MT v, const fr_t& x) {
  if constexpr (sizeof(MT) == 2)
    mac_u16(acc, (uint32_t)((int32_t)v + 32768), x);
  else
    mac_u64(acc, (uint64_t)v ^ 0x8000000000000000ull, x);
}

// row products, R rows per thread (x reused R times from one broadcast
// load): raw accumulator partials part[chunk][row][NW].  Split-K over column
// chunks gives the grid its parallelism; the epilogue is a plain store.
template <class MT, int R>
__global__ void __launch_bounds__(256)
    k_mvf_rows(const MT* M, uint64_t rows, uint64_t cols, const fr_t* x, uint64_t cch,
               uint64_t* part) {
  constexpr int CH = sizeof(MT) == 2 ? 1 : 4;
  constexpr int E = 64 / sizeof(MT);  // entries per 64-byte step (per row)
  using IO = AccIO<CH>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  fr_t* xs = reinterpret_cast<fr_t*>(smem_raw);
  const uint64_t c0 = blockIdx.y * cch;
  const uint64_t c1 = c0 + cch < cols ? c0 + cch : cols;
  const int n = (int)(c1 - c0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = x[c0 + i];
  __syncthreads();
  if (blockIdx.x == 0) chunk_sum_atomic(x, c0, n, part + rows * IO::NW);
  const uint64_t r0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * R;
  if (r0 >= rows) return;
  LimbAcc<CH> acc[R];
#pragma unroll
  for (int q = 0; q < R; q++) acc[q].zero();
  const MT* row0 = M + r0 * cols + c0;
  const bool full = r0 + R <= rows;
  int c = 0;
  if (full && ((uintptr_t)row0 % 16) == 0 && (cols * sizeof(MT)) % 16 == 0) {
    MT cur[R][E], nxt[R][E];
    auto load = [&](MT (&dst)[R][E], int at) {
#pragma unroll
      for (int q = 0; q < R; q++) {
        const uint4* p = reinterpret_cast<const uint4*>(row0 + q * cols + at);
#pragma unroll
        for (int h = 0; h < 4; h++) reinterpret_cast<uint4*>(dst[q])[h] = __ldcs(p + h);
      }
    };
    if (c + E <= n) load(cur, c);
    for (; c + E <= n; c += E) {
      const bool more = c + 2 * E <= n;
      if (more) load(nxt, c + E);  // software prefetch of the next step
#pragma unroll
      for (int k = 0; k < E; k++) {
        const fr_t xv = xs[c + k];
#pragma unroll
        for (int q = 0; q < R; q++) mac_entry<MT>(acc[q], cur[q][k], xv);
      }
      if (more) {
#pragma unroll
        for (int q = 0; q < R; q++)
#pragma unroll
          for (int k = 0; k < E; k++) cur[q][k] = nxt[q][k];
      }
    }
  }
  for (; c < n; c++) {
    const fr_t xv = xs[c];
#pragma unroll
    for (int q = 0; q < R; q++)
      if (r0 + q < rows) mac_entry<MT>(acc[q], row0[q * cols + c], xv);
  }
#pragma unroll
  for (int q = 0; q < R; q++)
    if (r0 + q < rows) IO::atomic_add(part + (r0 + q) * IO::NW, acc[q]);
}

// column products, thread per V consecutive columns: raw partials
// part[chunk][col][NW]; coalesced row segments, x[r] broadcast.
template <class MT, int V>
__global__ void __launch_bounds__(256)
    k_mvf_cols(const MT* M, uint64_t rows, uint64_t cols, const fr_t* x, uint64_t rch,
               uint64_t* part) {
  constexpr int CH = sizeof(MT) == 2 ? 1 : 4;
  using IO = AccIO<CH>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  fr_t* xs = reinterpret_cast<fr_t*>(smem_raw);
  const uint64_t r0 = blockIdx.y * rch;
  const uint64_t r1 = r0 + rch < rows ? r0 + rch : rows;
  const int n = (int)(r1 - r0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = x[r0 + i];
  __syncthreads();
  if (blockIdx.x == 0) chunk_sum_atomic(x, r0, n, part + cols * IO::NW);
  const uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * V;
  if (c >= cols) return;
  LimbAcc<CH> acc[V];
#pragma unroll
  for (int v = 0; v < V; v++) acc[v].zero();
  auto load = [&](MT (&vals)[V], int i) {
    const MT* p = M + (r0 + i) * cols + c;
    if constexpr (sizeof(MT) * V == 8) {
      *reinterpret_cast<uint2*>(vals) = __ldcs(reinterpret_cast<const uint2*>(p));
    } else if constexpr (sizeof(MT) * V == 16) {
      *reinterpret_cast<uint4*>(vals) = __ldcs(reinterpret_cast<const uint4*>(p));
    } else {
#pragma unroll
      for (int v = 0; v < V; v++) vals[v] = p[v];
    }
  };
  // batches of RB rows: RB independent loads in flight, next batch
  // prefetched while this one is multiplied (hides DRAM latency with few warps)
  constexpr int RB = 8;
  MT cur[RB][V], nxt[RB][V];
  auto load_batch = [&](MT (&dst)[RB][V], int at) {
#pragma unroll
    for (int b = 0; b < RB; b++) {
      if (at + b < n) load(dst[b], at + b);
      else {
#pragma unroll
        for (int v = 0; v < V; v++) dst[b][v] = 0;
      }
    }
  };
  if (n > 0) load_batch(cur, 0);
  for (int i = 0; i < n; i += RB) {
    const bool more = i + RB < n;
    if (more) load_batch(nxt, i + RB);
#pragma unroll
    for (int b = 0; b < RB; b++) {
      if (i + b < n) {
        const fr_t xv = xs[i + b];
#pragma unroll
        for (int v = 0; v < V; v++) mac_entry<MT>(acc[v], cur[b][v], xv);
      }
    }
    if (more) {
#pragma unroll
      for (int b = 0; b < RB; b++)
#pragma unroll
        for (int v = 0; v < V; v++) cur[b][v] = nxt[b][v];
    }
  }
#pragma unroll
  for (int v = 0; v < V; v++) IO::atomic_add(part + (c + v) * IO::NW, acc[v]);
}

// sum_{i<n} x[c0 + i] as a wide integer, added limb by limb into sumx[0..8]
// (u64, red.add) by warp 0 of one block per chunk: the offset-binary
// correction OFF * sum(x) is then formed by the finish kernel, no extra pass.
ZKL_D void chunk_sum_atomic(const fr_t* x, uint64_t c0, int n, uint64_t* sumx) {
  if ((threadIdx.x >> 5) != 0) return;
  const int lane = threadIdx.x & 31;
  uint64_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = lane; i < n; i += 32) {
    const fr_t v = x[c0 + i];
#pragma unroll
    for (int l = 0; l < 8; l++) acc[l] += v.v[l];  // <= 2^16 terms < 2^48
  }
#pragma unroll
  for (int l = 0; l < 8; l++) {
#pragma unroll
    for (int off = 16; off; off >>= 1) acc[l] += __shfl_xor_sync(kFull, acc[l], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int l = 0; l < 8; l++) atomicAdd((unsigned long long*)sumx + l, (unsigned long long)acc[l]);
  }
}

// Row products with lanes along COLUMNS (coalesced 256-byte row segments per
// warp), R rows per warp sharing each x load, x staged limb-major (SoA) so
// every lane's 16-byte shared load is conflict-free.  Per step a lane takes 4
// consecutive columns of R rows: 4R int16 entries, 32R mad.wide.  The lanes'
// raw u64 accumulators are summed with warp shuffles; lane 0 adds them to the
// row's record (red.add.u64: exact, order-free across column chunks).
template <int R>
__device__ __forceinline__ void mvw_rows_group(const int16_t* M, uint64_t rows,
                                                    uint64_t cols, const uint32_t* xsm,
                                                    uint64_t cch, int n, uint64_t c0,
                                                    uint64_t r0, int lane, uint64_t* acc_out) {
  LimbAcc<1> acc[R];
#pragma unroll
  for (int q = 0; q < R; q++) acc[q].zero();
  const int16_t* base = M + r0 * cols + c0;
  auto load = [&](uint2 (&dst)[R], int c) {
#pragma unroll
    for (int q = 0; q < R; q++)
      dst[q] = (r0 + q < rows && c < n)
                   ? __ldcs(reinterpret_cast<const uint2*>(base + q * cols + c))
                   : make_uint2(0, 0);
  };
  uint2 nxt[R];
  load(nxt, lane * 4);
  for (int c = lane * 4; c < n; c += 128) {
    uint2 mv[R];
#pragma unroll
    for (int q = 0; q < R; q++) mv[q] = nxt[q];
    load(nxt, c + 128);  // next step's entries in flight while this one multiplies
    uint4 xv[8];
#pragma unroll
    for (int l = 0; l < 8; l++) xv[l] = *reinterpret_cast<const uint4*>(xsm + l * cch + c);
#pragma unroll
    for (int v = 0; v < 4; v++) {
#pragma unroll
      for (int q = 0; q < R; q++) {
        const uint32_t word = v < 2 ? mv[q].x : mv[q].y;
        const int16_t sv = (int16_t)(v & 1 ? word >> 16 : word & 0xffffu);
        const uint32_t u = (uint32_t)((int32_t)sv + 32768);
#pragma unroll
        for (int l = 0; l < 8; l++) {
          const uint32_t xl = v == 0 ? xv[l].x : v == 1 ? xv[l].y : v == 2 ? xv[l].z : xv[l].w;
          acc[q].e[l] = madw(u, xl, acc[q].e[l]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < R; q++) {
#pragma unroll
    for (int l = 0; l < 8; l++) {
      uint64_t t = acc[q].e[l];
#pragma unroll
      for (int off = 16; off; off >>= 1) t += __shfl_xor_sync(kFull, t, off);
      acc[q].e[l] = t;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < R; q++)
      if (r0 + q < rows) AccIO<1>::atomic_add(acc_out + (r0 + q) * 8, acc[q]);
  }
}

template <int R>
__global__ void __launch_bounds__(256, (R == 2 ? 3 : 2))
    k_mvw_rows(const int16_t* M, uint64_t rows, uint64_t cols, const fr_t* x, uint64_t cch,
               uint64_t* acc_out) {
  extern __shared__ __align__(16) uint32_t xsm[];  // 8 limbs x cch
  const uint64_t c0 = blockIdx.y * cch;
  const int n = (int)((c0 + cch < cols ? c0 + cch : cols) - c0);
  // stage x: every thread issues all of its loads before the first store
  // (one L2 round trip instead of one per element)
  constexpr int kFill = 8;  // cch <= 8 * 256
  fr_t xr[kFill];
#pragma unroll
  for (int k = 0; k < kFill; k++) {
    const int i = threadIdx.x + k * 256;
    if (i < n) xr[k] = x[c0 + i];
  }
#pragma unroll
  for (int k = 0; k < kFill; k++) {
    const int i = threadIdx.x + k * 256;
    if (i < n) {
#pragma unroll
      for (int l = 0; l < 8; l++) xsm[l * cch + i] = xr[k].v[l];
    }
  }
  __syncthreads();
  if (blockIdx.x == 0) chunk_sum_atomic(x, c0, n, acc_out + rows * 8);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the block's x chunk is staged once and reused for every row group the
  // block's warps take (grid-stride over rows)
  const uint64_t rstride = (uint64_t)gridDim.x * (blockDim.x >> 5) * R;
  for (uint64_t r0 = (blockIdx.x * (uint64_t)(blockDim.x >> 5) + warp) * R; r0 < rows;
       r0 += rstride)
    mvw_rows_group<R>(M, rows, cols, xsm, cch, n, c0, r0, lane, acc_out);
}

// Tensor-core int16 row products (mma.sync m16n8k32 u8 x u8 -> s32).  The
// field vector is split into its 32 bytes and each offset-binary entry
// u = s + 2^15 into two bytes, so y_r = sum_c u_rc x_c is
//   sum_{s in lo,hi} sum_{n < 32} 2^(8(n+s)) * (sum_c u_s[r][c] x_n[c]),
// a 16-row x 32-byte x K GEMM per warp whose int32 outputs are exact (each
// < 255 * 255 * K, K <= 256 per chunk).  The byte sums are folded into the
// same per-limb u64 row records as k_mvw_rows (limb b/4, shift 8 (b % 4);
// the top byte b = 32 goes to limb 7 << 32), so k_mvf_finish and the
// OFF * sum(x) correction are shared.  x is staged as 32 byte planes with a
// 16-byte skew per plane (conflict-free B-fragment loads); the integer pipe
// then only assembles fragments: the IMAD-bound MAC loop becomes a load
// stream.
#ifndef ZKL_TCK
#define ZKL_TCK 256
#endif
#ifndef ZKL_TCK_MINB
#define ZKL_TCK_MINB 1
#endif
constexpr int kTcK = ZKL_TCK;  // columns per chunk: kTcK / 32 k-steps, all loads issued up front

ZKL_D void mma_u8(uint32_t (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(256, ZKL_TCK_MINB)
    k_mvt_rows(const int16_t* M, uint64_t rows, uint64_t cols, const fr_t* x,
               uint64_t* acc_out) {
  // plane stride: a 32-byte skew keeps the per-half-warp 8-byte B loads
  // (plane 8t + g, offset 8 tig) on distinct banks
  constexpr int PS = kTcK + 32;
  constexpr int kSteps = kTcK / 32;
  extern __shared__ __align__(16) uint8_t planes[];  // 32 x PS
  const uint64_t c0 = blockIdx.y * (uint64_t)kTcK;
  const int n = (int)((c0 + kTcK < cols ? c0 + kTcK : cols) - c0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const uint64_t r0 = (blockIdx.x * 8ull + warp) * 16;
  const bool active = r0 < rows;
  // The reduction order over k is free, so each thread's A fragment holds the
  // 8 consecutive columns it loads with one 16-byte load per row (k slots
  // tig*4..+3 <- columns 8 tig..+3, slots 16 + tig*4.. <- 8 tig + 4..7), and
  // its B fragment is the matching 8 bytes of one x byte plane.  The warp's
  // whole 16 x kTcK tile is requested first, so its latency overlaps the x
  // staging below.
  const int16_t* rowA = M + (r0 + g) * cols + c0 + tig * 8;
  const int16_t* rowB = rowA + 8 * cols;
  uint4 buf[kSteps][2];
#pragma unroll
  for (int st = 0; st < kSteps; st++) {
    const int k = st * 32;
    if (active && k < n) {
      buf[st][0] = __ldcs(reinterpret_cast<const uint4*>(rowA + k));
      buf[st][1] = __ldcs(reinterpret_cast<const uint4*>(rowB + k));
    }
  }
  // stage x[c0 .. c0+n) as byte planes: a thread takes 4 consecutive elements
  for (int j4 = threadIdx.x * 4; j4 < n; j4 += blockDim.x * 4) {
    uint32_t w[4][8];
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const fr_t v = j4 + e < n ? x[c0 + j4 + e] : fr_t{};
#pragma unroll
      for (int l = 0; l < 8; l++) w[e][l] = v.v[l];
    }
#pragma unroll
    for (int l = 0; l < 8; l++) {
#pragma unroll
      for (int b = 0; b < 4; b++) {
        // byte b of limb l of the 4 elements -> plane 4l+b, offset j4
        const uint32_t lo = __byte_perm(w[0][l], w[1][l], 0x0040 + b * 0x0011) & 0xffffu;
        const uint32_t hi = __byte_perm(w[2][l], w[3][l], 0x0040 + b * 0x0011) & 0xffffu;
        *reinterpret_cast<uint32_t*>(planes + (4 * l + b) * PS + j4) = lo | (hi << 16);
      }
    }
  }
  __syncthreads();
  if (blockIdx.x == 0) chunk_sum_atomic(x, c0, n, acc_out + rows * 8);
  if (!active) return;
  uint32_t acc[2][4][4];
#pragma unroll
  for (int sl = 0; sl < 2; sl++)
#pragma unroll
    for (int t = 0; t < 4; t++)
#pragma unroll
      for (int q = 0; q < 4; q++) acc[sl][t][q] = 0;
#pragma unroll
  for (int st = 0; st < kSteps; st++) {
    const int k = st * 32;
    if (k >= n) break;
    uint32_t alo[4], ahi[4];
    // a0 / a2: row g, columns 8 tig + 0..3 / 4..7; a1 / a3: row g + 8.
    // Offset binary: flip each int16's sign bit.
    const uint4 ra = buf[st][0], rb = buf[st][1];
    const uint32_t wa[4] = {ra.x ^ 0x80008000u, ra.y ^ 0x80008000u, ra.z ^ 0x80008000u,
                            ra.w ^ 0x80008000u};
    const uint32_t wb[4] = {rb.x ^ 0x80008000u, rb.y ^ 0x80008000u, rb.z ^ 0x80008000u,
                            rb.w ^ 0x80008000u};
    alo[0] = __byte_perm(wa[0], wa[1], 0x6420);
    ahi[0] = __byte_perm(wa[0], wa[1], 0x7531);
    alo[1] = __byte_perm(wb[0], wb[1], 0x6420);
    ahi[1] = __byte_perm(wb[0], wb[1], 0x7531);
    alo[2] = __byte_perm(wa[2], wa[3], 0x6420);
    ahi[2] = __byte_perm(wa[2], wa[3], 0x7531);
    alo[3] = __byte_perm(wb[2], wb[3], 0x6420);
    ahi[3] = __byte_perm(wb[2], wb[3], 0x7531);
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const uint2 bb =
          *reinterpret_cast<const uint2*>(planes + (8 * t + g) * PS + k + tig * 8);
      mma_u8(acc[0][t], alo, bb.x, bb.y);
      mma_u8(acc[1][t], ahi, bb.x, bb.y);
    }
  }
  // fold byte sums into per-limb records for rows g and g + 8: the sum for
  // byte position b = 8t + rel (rel = 2 tig + (q & 1) + slice, 0..8) goes to
  // limb 2t + (rel >> 2) shifted by 8 (rel & 3); b = 32 goes to limb 7 << 32
  uint64_t e[2][8];
#pragma unroll
  for (int h = 0; h < 2; h++)
#pragma unroll
    for (int l = 0; l < 8; l++) e[h][l] = 0;
#pragma unroll
  for (int sl = 0; sl < 2; sl++)
#pragma unroll
    for (int t = 0; t < 4; t++)
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int h = q >> 1;  // c0, c1: row g; c2, c3: row g + 8
        const int rel = 2 * tig + (q & 1) + sl;
        const uint64_t v = (uint64_t)acc[sl][t][q] << (8 * (rel & 3));
        const int off = rel >> 2;
        e[h][2 * t] += off == 0 ? v : 0;
        e[h][2 * t + 1] += off == 1 ? v : 0;
        if (t < 3) e[h][2 * t + 2] += off == 2 ? v : 0;
        else e[h][7] += off == 2 ? ((uint64_t)acc[sl][t][q] << 32) : 0;
      }
#pragma unroll
  for (int h = 0; h < 2; h++)
#pragma unroll
    for (int l = 0; l < 8; l++) {
      e[h][l] += __shfl_xor_sync(kFull, e[h][l], 1);
      e[h][l] += __shfl_xor_sync(kFull, e[h][l], 2);
    }
  if (tig == 0) {
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint64_t r = r0 + g + 8 * h;
      if (r < rows) {
        unsigned long long* d = reinterpret_cast<unsigned long long*>(acc_out + r * 8);
#pragma unroll
        for (int l = 0; l < 8; l++) atomicAdd(d + l, (unsigned long long)e[h][l]);
      }
    }
  }
}

// Tensor-core int16 COLUMN products y_c = sum_r M[r][c] x_r (M^T x), the
// same byte-sliced GEMM as k_mvt_rows with the roles of the operands swapped:
//   D[byte m][col c] = sum_r X[m][r] * U_slice[r][c]   (m16n8k32, u8 x u8),
// A = the 32 byte planes of x (two 16-byte m-tiles), B = a slice of the
// offset-binary matrix.  A block stages a 256-row x 128-column tile of M
// row-major in shared memory (coalesced 16-byte loads); ldmatrix.trans
// hands each thread M[8i + 2 tig + {0,1}][c0 + g] for the four 8-row groups
// i, so the k slots of both fragments follow the permutation
//   slot tig*4 + 2i' + j  <->  row 8 i' + 2 tig + j      (i' = 0, 1)
//   slot 16 + tig*4 + 2i' + j <-> row 16 + 8 i' + 2 tig + j,
// and x is staged into its byte planes in that slot order (one LDS.32 per A
// register).  Each warp owns 16 columns (two n-tiles); the byte sums are
// folded into the shared per-limb column records.
constexpr int kTcR = 256;          // rows per block (K)
constexpr int kTcC = 128;          // columns per block (8 warps x 16)
constexpr int kTcMP = kTcC * 2 + 16;  // smem row pitch of the M tile (bytes)

ZKL_D int slot_of_row(int r) {  // r in [0, 32): k slot of row r
  const int half = r >> 4, rr = r & 15;
  const int i = rr >> 3, t = (rr & 7) >> 1, j = r & 1;
  return half * 16 + t * 4 + 2 * i + j;
}

__global__ void __launch_bounds__(256)
    k_mvt_cols(const int16_t* M, uint64_t rows, uint64_t cols, const fr_t* x,
               uint64_t* acc_out) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint8_t* mt = sm;                           // kTcR x kTcMP bytes
  uint8_t* planes = sm + kTcR * kTcMP;        // 32 x (kTcR + 16)
  constexpr int XP = kTcR + 16;
  const uint64_t r0 = blockIdx.y * (uint64_t)kTcR;
  const uint64_t c0 = blockIdx.x * (uint64_t)kTcC;
  const int nr = (int)((r0 + kTcR < rows ? r0 + kTcR : rows) - r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tig = lane & 3;
  // stage the M tile (row-major, offset binary applied at fragment time)
  {
    constexpr int kPerRow = kTcC / 8;  // uint4 per tile row
    uint4 v[kTcR * kPerRow / 256];
#pragma unroll
    for (int q = 0; q < kTcR * kPerRow / 256; q++) {
      const int idx = threadIdx.x + q * 256;
      const int r = idx / kPerRow, cq = idx % kPerRow;
      v[q] = (r < nr && c0 + cq * 8 < cols)
                 ? __ldcs(reinterpret_cast<const uint4*>(M + (r0 + r) * cols + c0 + cq * 8))
                 : make_uint4(0x80008000u, 0x80008000u, 0x80008000u, 0x80008000u);
    }
#pragma unroll
    for (int q = 0; q < kTcR * kPerRow / 256; q++) {
      const int idx = threadIdx.x + q * 256;
      const int r = idx / kPerRow, cq = idx % kPerRow;
      *reinterpret_cast<uint4*>(mt + r * kTcMP + cq * 16) = v[q];
    }
  }
  // stage x[r0 .. r0+nr) as byte planes in k-slot order (4 elements a thread)
  for (int j4 = threadIdx.x * 4; j4 < kTcR; j4 += blockDim.x * 4) {
    uint32_t w[4][8];
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const fr_t v = j4 + e < nr ? x[r0 + j4 + e] : fr_t{};
#pragma unroll
      for (int l = 0; l < 8; l++) w[e][l] = v.v[l];
    }
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int r = j4 + e;
      const int pos = (r & ~31) + slot_of_row(r & 31);
#pragma unroll
      for (int l = 0; l < 8; l++)
#pragma unroll
        for (int b = 0; b < 4; b++) planes[(4 * l + b) * XP + pos] = (uint8_t)(w[e][l] >> (8 * b));
    }
  }
  __syncthreads();
  if (blockIdx.x == 0) chunk_sum_atomic(x, r0, nr, acc_out + cols * 8);
  const uint64_t wc = c0 + warp * 16;  // this warp's 16 columns
  if (wc >= cols) return;
  uint32_t acc[2][2][2][4];  // [m-tile][n-tile][slice][frag]
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 2; b++)
#pragma unroll
      for (int sl = 0; sl < 2; sl++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[a][b][sl][q] = 0;
  const uint32_t mt_base = (uint32_t)__cvta_generic_to_shared(mt);
  for (int k = 0; k < nr; k += 32) {
    // A: x byte planes, rows in slot order: a0 / a2 plane m at slots tig*4 /
    // 16 + tig*4, a1 / a3 plane m + 8
    uint32_t afr[2][4];
#pragma unroll
    for (int mtile = 0; mtile < 2; mtile++) {
      const uint8_t* p0 = planes + (16 * mtile + g) * XP + k + tig * 4;
      const uint8_t* p1 = p0 + 8 * XP;
      afr[mtile][0] = *reinterpret_cast<const uint32_t*>(p0);
      afr[mtile][1] = *reinterpret_cast<const uint32_t*>(p1);
      afr[mtile][2] = *reinterpret_cast<const uint32_t*>(p0 + 16);
      afr[mtile][3] = *reinterpret_cast<const uint32_t*>(p1 + 16);
    }
#pragma unroll
    for (int nt = 0; nt < 2; nt++) {
      // ldmatrix.x4.trans: matrix i = rows k + 8i .. +7, columns wc + 8 nt .. +7
      const int row = k + lane;  // lanes 8i..8i+7 address matrix i's rows
      const uint32_t addr = mt_base + row * kTcMP + (uint32_t)((wc - c0) + 8 * nt) * 2;
      uint32_t m0, m1, m2, m3;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(m0), "=r"(m1), "=r"(m2), "=r"(m3) : "r"(addr));
      m0 ^= 0x80008000u; m1 ^= 0x80008000u; m2 ^= 0x80008000u; m3 ^= 0x80008000u;
      // b0: rows 2tig+{0,1} (m0), 8+2tig+{0,1} (m1); b1: the same 16 rows on
      const uint32_t blo0 = __byte_perm(m0, m1, 0x6420), bhi0 = __byte_perm(m0, m1, 0x7531);
      const uint32_t blo1 = __byte_perm(m2, m3, 0x6420), bhi1 = __byte_perm(m2, m3, 0x7531);
#pragma unroll
      for (int mtile = 0; mtile < 2; mtile++) {
        mma_u8(acc[mtile][nt][0], afr[mtile], blo0, blo1);
        mma_u8(acc[mtile][nt][1], afr[mtile], bhi0, bhi1);
      }
    }
  }
  // fold: lane (g, tig) holds, for columns 2 tig, 2 tig + 1 of each n-tile,
  // the byte sums of bytes m = g, g + 8 (m-tile 0) and g + 16, g + 24
  uint64_t e[2][2][8];  // [n-tile][column parity][limb]
#pragma unroll
  for (int nt = 0; nt < 2; nt++)
#pragma unroll
    for (int cp = 0; cp < 2; cp++)
#pragma unroll
      for (int l = 0; l < 8; l++) e[nt][cp][l] = 0;
#pragma unroll
  for (int mtile = 0; mtile < 2; mtile++)
#pragma unroll
    for (int nt = 0; nt < 2; nt++)
#pragma unroll
      for (int sl = 0; sl < 2; sl++)
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int cp = q & 1;
          const int mrel = 16 * mtile + 8 * (q >> 1);  // byte = g + mrel
          const int bpos = g + mrel + sl;              // 0 .. 32
          const int l = bpos >> 2;                     // runtime (g): select below
          const uint64_t v = (uint64_t)acc[mtile][nt][sl][q] << (8 * (bpos & 3));
#pragma unroll
          for (int ll = 0; ll < 8; ll++) {
            // bpos 32 (g = 7, top m-tile row 24, hi slice) -> limb 7 << 32
            const uint64_t add = (ll == 7 && bpos == 32) ? ((uint64_t)acc[mtile][nt][sl][q] << 32)
                                 : (l == ll ? v : 0);
            e[nt][cp][ll] += add;
          }
        }
#pragma unroll
  for (int nt = 0; nt < 2; nt++)
#pragma unroll
    for (int cp = 0; cp < 2; cp++)
#pragma unroll
      for (int l = 0; l < 8; l++) {
        uint64_t t = e[nt][cp][l];
        t += __shfl_xor_sync(kFull, t, 4);
        t += __shfl_xor_sync(kFull, t, 8);
        t += __shfl_xor_sync(kFull, t, 16);
        e[nt][cp][l] = t;
      }
  if (g == 0) {
#pragma unroll
    for (int nt = 0; nt < 2; nt++)
#pragma unroll
      for (int cp = 0; cp < 2; cp++) {
        const uint64_t c = wc + 8 * nt + 2 * tig + cp;
        if (c < cols) {
          unsigned long long* d = reinterpret_cast<unsigned long long*>(acc_out + c * 8);
#pragma unroll
          for (int l = 0; l < 8; l++) atomicAdd(d + l, (unsigned long long)e[nt][cp][l]);
        }
      }
  }
}

// y[i] = reduce(acc[i]) - K; one thread per output (acc: atomically summed
// raw words of every chunk -- exact integer sums, order-independent)
template <int CH>
__global__ void __launch_bounds__(256)
    k_mvf_finish(const uint64_t* part, uint64_t n, const uint64_t* sumx, fr_t offr, fr_t* y) {
  using IO = AccIO<CH>;
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  // K = OFF * sum(x) mod p (sumx: 8 u64 limb sums), by every thread: no
  // barrier, and the chain overlaps the thread's own reduction
  LimbAcc<1> sa;
#pragma unroll
  for (int l = 0; l < 8; l++) sa.e[l] = sumx[l];
  const fr_t s_k = Fr255::mul(limb_reduce<1>(sa), offr);
  LimbAcc<CH> acc;
  acc.zero();
  IO::add(acc, part + i * IO::NW);
  y[i] = Fr255::sub(limb_reduce<CH>(acc), s_k);
}

// ---------------------------------------------------------------------------
// Tensor-core int64 products (the zkMat C operands).  Each entry's offset-
// binary value u = s + 2^63 is split into its 8 bytes (planes p = 0..7) and x
// into its 32 bytes, so
//   sum_c u_c x_c = sum_{p, m} 2^(8(p+m)) sum_c U_p[c] X_m[c],
// one u8 x u8 GEMM per plane with M = the 32 x bytes (two m16 tiles, the A
// operand from shared byte planes) and N = 8 matrix rows / columns per warp
// (the B operand).  Every int32 sum is exact: < 255 * 255 * 512 < 2^25 per
// 512-entry chunk.  The epilogue adds each lane's sums into per-position
// totals in shared memory (position b = p + m, 39 of them per output), folds
// them into ten 32-bit-spaced u64 limbs and red.adds those into the output's
// record; k_mvt64_finish reduces the record mod p and subtracts
// 2^63 * sum(x).  Per entry: one 8-byte load, 2 byte permutes, 16/32 MMA
// slots -- the 32 carry-chained IMAD.WIDE of the wide-accumulator kernel
// become a load stream.
constexpr int kT64K = 512;             // entries of the reduction dimension per block
constexpr int kT64Steps = kT64K / 32;  // k-steps of 32
constexpr int kT64XP = kT64K + 16;     // x plane pitch (bytes)
constexpr int kT64NW = 10;             // u64 limbs per output record

// x[k0 .. k0+n) -> 32 byte planes (plane m holds byte m of every element),
// zero past n; 128 threads, 4 elements each
ZKL_D void t64_stage_x(const fr_t* x, uint64_t k0, int n, uint8_t* planes) {
  for (int j4 = threadIdx.x * 4; j4 < kT64K; j4 += blockDim.x * 4) {
    uint32_t w[4][8];
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const fr_t v = j4 + e < n ? x[k0 + j4 + e] : fr_t{};
#pragma unroll
      for (int l = 0; l < 8; l++) w[e][l] = v.v[l];
    }
#pragma unroll
    for (int l = 0; l < 8; l++) {
#pragma unroll
      for (int b = 0; b < 4; b++) {
        const uint32_t lo = __byte_perm(w[0][l], w[1][l], 0x0040 + b * 0x0011) & 0xffffu;
        const uint32_t hi = __byte_perm(w[2][l], w[3][l], 0x0040 + b * 0x0011) & 0xffffu;
        *reinterpret_cast<uint32_t*>(planes + (4 * l + b) * kT64XP + j4) = lo | (hi << 16);
      }
    }
  }
}

// four int64 entries (words lo/hi) -> the 8 byte-plane registers of one B
// half-fragment: reg p = byte p of e0..e3 (offset binary on plane 7)
ZKL_D void t64_planes(const uint32_t (&lo)[4], const uint32_t (&hi)[4], uint32_t (&b)[8]) {
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const uint32_t* w = h ? hi : lo;
#pragma unroll
    for (int q = 0; q < 2; q++) {  // planes 4h + 2q, 4h + 2q + 1
      const uint32_t sel = (uint32_t)((2 * q) | ((2 * q + 4) << 4) | ((2 * q + 1) << 8) |
                                      ((2 * q + 5) << 12));
      const uint32_t t01 = __byte_perm(w[0], w[1], sel);  // e0.p, e1.p, e0.p+1, e1.p+1
      const uint32_t t23 = __byte_perm(w[2], w[3], sel);
      b[4 * h + 2 * q] = __byte_perm(t01, t23, 0x5410);
      b[4 * h + 2 * q + 1] = __byte_perm(t01, t23, 0x7632);
    }
  }
  b[7] ^= 0x80808080u;
}

// MMAs of one k-step: acc[p][mt] += X_planes(mt) x U_p
ZKL_D void t64_mma(uint32_t (&acc)[8][2][4], const uint8_t* planes, int ks, int g, int tig,
                   const uint32_t (&b0)[8], const uint32_t (&b1)[8]) {
  uint32_t afr[2][4];
#pragma unroll
  for (int mt = 0; mt < 2; mt++) {
    const uint8_t* p0 = planes + (16 * mt + g) * kT64XP + ks * 32 + tig * 4;
    const uint8_t* p1 = p0 + 8 * kT64XP;
    afr[mt][0] = *reinterpret_cast<const uint32_t*>(p0);
    afr[mt][1] = *reinterpret_cast<const uint32_t*>(p1);
    afr[mt][2] = *reinterpret_cast<const uint32_t*>(p0 + 16);
    afr[mt][3] = *reinterpret_cast<const uint32_t*>(p1 + 16);
  }
#pragma unroll
  for (int p = 0; p < 8; p++)
#pragma unroll
    for (int mt = 0; mt < 2; mt++) mma_u8(acc[p][mt], afr[mt], b0[p], b1[p]);
}

// epilogue: lane (g, tig) holds D[m][n] for x bytes m = 16 mt + g (+ 8) and
// outputs n = 2 tig, 2 tig + 1 of the warp's 8; position sums in shared
// memory (distinct addresses per instruction), then limbs -> red.add
ZKL_D void t64_epilogue(const uint32_t (&acc)[8][2][4], uint32_t* pos /* 8 x 40 */, int lane,
                        int g, int tig, uint64_t out0, uint64_t nout, uint64_t* rec) {
  for (int i = lane; i < 8 * 40; i += 32) pos[i] = 0;
  __syncwarp();
#pragma unroll
  for (int p = 0; p < 8; p++)
#pragma unroll
    for (int mt = 0; mt < 2; mt++)
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int m = 16 * mt + g + 8 * (q >> 1), n = 2 * tig + (q & 1);
        atomicAdd(pos + n * 40 + m + p, acc[p][mt][q]);
      }
  __syncwarp();
  for (int i = lane; i < 8 * kT64NW; i += 32) {
    const int n = i / kT64NW, L = i % kT64NW;
    const uint32_t* P = pos + n * 40 + 4 * L;
    const uint64_t v = (uint64_t)P[0] + ((uint64_t)P[1] << 8) + ((uint64_t)P[2] << 16) +
                       ((uint64_t)P[3] << 24);
    if (out0 + n < nout && v)
      atomicAdd(reinterpret_cast<unsigned long long*>(rec + (out0 + n) * kT64NW + L),
                (unsigned long long)v);
  }
}

// y_r = sum_c M[r][c] x_c: grid (rows / 32, ceil(cols / 512)), 4 warps x 8 rows
__global__ void __launch_bounds__(128)
    k_mvt64_rows(const int64_t* M, uint64_t rows, uint64_t cols, const fr_t* x, uint64_t* rec) {
  __shared__ __align__(16) uint8_t planes[32 * kT64XP];
  __shared__ uint32_t pos[4][8 * 40];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const uint64_t k0 = blockIdx.y * (uint64_t)kT64K;
  const int n = (int)((k0 + kT64K < cols ? k0 + kT64K : cols) - k0);
  const uint64_t r0 = blockIdx.x * 32ull + warp * 8;
  const uint64_t row = r0 + g;
  const bool live = row < rows;
  const int64_t* base = M + (live ? row : 0) * cols + k0 + tig * 4;
  // entries for k-step ks: columns 4 tig .. +3 and 16 + 4 tig .. +3 (32 B each)
  auto load = [&](uint4 (&d)[4], int ks) {
    const int c = ks * 32;
    if (live && c + 32 <= n) {
      const uint4* p = reinterpret_cast<const uint4*>(base + c);
      d[0] = __ldcs(p);
      d[1] = __ldcs(p + 1);
      d[2] = __ldcs(p + 8);
      d[3] = __ldcs(p + 9);
    } else {
      // ragged tail: u = 0 contributes nothing after the 2^63 correction,
      // so pad with s = -2^63 (u = 0) and with x = 0 in the planes
#pragma unroll
      for (int h = 0; h < 4; h++) {
        const int cc = c + (h >> 1) * 16 + tig * 4 + (h & 1) * 2;
        int64_t v0 = (int64_t)0x8000000000000000ull, v1 = v0;
        if (live && cc < n) v0 = base[c + (h >> 1) * 16 + (h & 1) * 2];
        if (live && cc + 1 < n) v1 = base[c + (h >> 1) * 16 + (h & 1) * 2 + 1];
        d[h] = make_uint4((uint32_t)v0, (uint32_t)((uint64_t)v0 >> 32), (uint32_t)v1,
                          (uint32_t)((uint64_t)v1 >> 32));
      }
    }
  };
  uint4 cur[4], nxt[4];
  load(cur, 0);
  t64_stage_x(x, k0, n, planes);
  __syncthreads();
  if (blockIdx.x == 0) chunk_sum_atomic(x, k0, n, rec + rows * kT64NW);
  uint32_t acc[8][2][4];
#pragma unroll
  for (int p = 0; p < 8; p++)
#pragma unroll
    for (int mt = 0; mt < 2; mt++)
#pragma unroll
      for (int q = 0; q < 4; q++) acc[p][mt][q] = 0;
  const int steps = (n + 31) / 32;
  for (int ks = 0; ks < steps; ks++) {
    if (ks + 1 < steps) load(nxt, ks + 1);
    uint32_t lo[4], hi[4], b0[8], b1[8];
    lo[0] = cur[0].x; hi[0] = cur[0].y; lo[1] = cur[0].z; hi[1] = cur[0].w;
    lo[2] = cur[1].x; hi[2] = cur[1].y; lo[3] = cur[1].z; hi[3] = cur[1].w;
    t64_planes(lo, hi, b0);
    lo[0] = cur[2].x; hi[0] = cur[2].y; lo[1] = cur[2].z; hi[1] = cur[2].w;
    lo[2] = cur[3].x; hi[2] = cur[3].y; lo[3] = cur[3].z; hi[3] = cur[3].w;
    t64_planes(lo, hi, b1);
    t64_mma(acc, planes, ks, g, tig, b0, b1);
#pragma unroll
    for (int h = 0; h < 4; h++) cur[h] = nxt[h];
  }
  t64_epilogue(acc, pos[warp], lane, g, tig, r0, rows, rec);
}

// y_c = sum_r M[r][c] x_r: grid (cols / 32, ceil(rows / 512)), 4 warps x 8
// columns; each k-step's 32 x 32 entry tile is staged in shared memory
// (coalesced 16-byte loads, 272-byte row pitch: the four tig groups' 8-byte
// column reads land on distinct banks)
constexpr int kT64TP = 32 * 8 + 16;  // tile row pitch (bytes)

__global__ void __launch_bounds__(128)
    k_mvt64_cols(const int64_t* M, uint64_t rows, uint64_t cols, const fr_t* x, uint64_t* rec) {
  __shared__ __align__(16) uint8_t planes[32 * kT64XP];
  __shared__ __align__(16) uint8_t tile[2][32 * kT64TP];
  __shared__ uint32_t pos[4][8 * 40];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const uint64_t k0 = blockIdx.y * (uint64_t)kT64K;  // first row of the chunk
  const int n = (int)((k0 + kT64K < rows ? k0 + kT64K : rows) - k0);
  const uint64_t c0 = blockIdx.x * 32ull;
  // tile load: thread t takes rows t / 16 + 8 i (i < 4), 16 bytes at column pair 2 (t % 16)
  const int tr = threadIdx.x >> 4, tc = (threadIdx.x & 15) * 2;
  auto load = [&](uint4 (&d)[4], int ks) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int r = ks * 32 + tr + 8 * i;
      const uint64_t cc = c0 + tc;
      if (r < n && cc + 1 < cols) {
        d[i] = __ldcs(reinterpret_cast<const uint4*>(M + (k0 + r) * cols + cc));
      } else {
        const int64_t pad = (int64_t)0x8000000000000000ull;  // u = 0
        const int64_t v0 = r < n && cc < cols ? M[(k0 + r) * cols + cc] : pad;
        d[i] = make_uint4((uint32_t)v0, (uint32_t)((uint64_t)v0 >> 32), (uint32_t)pad,
                          (uint32_t)((uint64_t)pad >> 32));
      }
    }
  };
  auto stash = [&](const uint4 (&d)[4], uint8_t* t) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      *reinterpret_cast<uint4*>(t + (tr + 8 * i) * kT64TP + tc * 8) = d[i];
  };
  uint4 cur[4];
  load(cur, 0);
  t64_stage_x(x, k0, n, planes);
  stash(cur, tile[0]);
  __syncthreads();
  if (blockIdx.x == 0) chunk_sum_atomic(x, k0, n, rec + cols * kT64NW);
  uint32_t acc[8][2][4];
#pragma unroll
  for (int p = 0; p < 8; p++)
#pragma unroll
    for (int mt = 0; mt < 2; mt++)
#pragma unroll
      for (int q = 0; q < 4; q++) acc[p][mt][q] = 0;
  const int steps = (n + 31) / 32;
  const int col = warp * 8 + g;  // this lane's column within the tile
  for (int ks = 0; ks < steps; ks++) {
    const bool more = ks + 1 < steps;
    if (more) load(cur, ks + 1);
    const uint8_t* t = tile[ks & 1];
    uint32_t lo[4], hi[4], b0[8], b1[8];
#pragma unroll
    for (int h = 0; h < 2; h++) {
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const uint2 v = *reinterpret_cast<const uint2*>(t + (16 * h + 4 * tig + i) * kT64TP + col * 8);
        lo[i] = v.x;
        hi[i] = v.y;
      }
      t64_planes(lo, hi, h ? b1 : b0);
    }
    t64_mma(acc, planes, ks, g, tig, b0, b1);
    if (more) stash(cur, tile[(ks + 1) & 1]);
    __syncthreads();
  }
  t64_epilogue(acc, pos[warp], lane, g, tig, c0 + warp * 8, cols, rec);
}

// y[i] = reduce(sum_L rec[i][L] 2^(32 L)) - 2^63 sum(x)
__global__ void __launch_bounds__(256)
    k_mvt64_finish(const uint64_t* rec, uint64_t n, const uint64_t* sumx, fr_t offr, fr_t* y) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  // K = 2^63 sum(x) mod p, by every thread (no barrier: this chain runs
  // beside the thread's own reduction)
  LimbAcc<1> sa;
#pragma unroll
  for (int l = 0; l < 8; l++) sa.e[l] = sumx[l];
  const fr_t s_k = Fr255::mul(limb_reduce<1>(sa), offr);
  // u64 limbs at 32-bit spacing -> 12 words with carries
  uint32_t w[12];
  uint64_t carry = 0;
#pragma unroll
  for (int j = 0; j < 12; j++) {
    uint64_t t = carry;
    if (j < kT64NW) t += (uint32_t)rec[i * kT64NW + j];
    if (j >= 1 && j - 1 < kT64NW) t += rec[i * kT64NW + j - 1] >> 32;
    w[j] = (uint32_t)t;
    carry = t >> 32;
  }
  fr_t lo, hi = Fr255::zero();
#pragma unroll
  for (int j = 0; j < 8; j++) lo.v[j] = w[j];
#pragma unroll
  for (int j = 8; j < 12; j++) hi.v[j - 8] = w[j];
  lo = Fr255::reduce_once(Fr255::reduce_once(lo));
  hi = Fr255::mul(hi, Fr255::r2());
  y[i] = Fr255::sub(Fr255::add(lo, hi), s_k);
}

static bool t64_enabled() {
  static const bool on = [] {
    const char* e = getenv("ZKL_MV_TC64");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// int64 matrix x Fr vector on the tensor cores; kErrUnsupported when the
// reduction dimension exceeds the record headroom
static int matvec_t64(const int64_t* M, uint64_t rows, uint64_t cols, int transpose,
                      const fr_t* x, fr_t* y, cudaStream_t s) {
  const uint64_t klen = transpose ? rows : cols, nout = transpose ? cols : rows;
  // limb headroom: ceil(klen / 512) <= 2^11 chunks x < 2^53 each stays below
  // 2^64; 16-byte loads need an even row length and an aligned base
  if (klen > (1ull << 20) || (cols & 1) || ((uintptr_t)M & 15)) return kErrUnsupported;
  void* ws;
  const size_t bytes = (nout * kT64NW + 8) * 8;
  int rc = scratch_reserve(bytes + 64, &ws, s);
  if (rc) return rc;
  ZKL_CUDA(cudaMemsetAsync(ws, 0, bytes, s));
  uint64_t* rec = (uint64_t*)ws;
  dim3 g((unsigned)((nout + 31) / 32), (unsigned)((klen + kT64K - 1) / kT64K));
  if (transpose)
    k_mvt64_cols<<<g, 128, 0, s>>>(M, rows, cols, x, rec);
  else
    k_mvt64_rows<<<g, 128, 0, s>>>(M, rows, cols, x, rec);
  ZKL_LAUNCH_CHECK();
  static fr_t offr = [] {
    fr_t v = Fr255::zero();
    v.v[1] = 1u << 31;  // 2^63
    return Fr255::to_mont(v);
  }();
  k_mvt64_finish<<<(unsigned)((nout + 255) / 256), 256, 0, s>>>(rec, nout, rec + nout * kT64NW,
                                                                 offr, y);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

// returns kErrUnsupported when the shape does not suit the fast kernels
template <class MT>
static int matvec_fast(const MT* M, uint64_t rows, uint64_t cols, int transpose, const fr_t* x,
                       fr_t* y, cudaStream_t s) {
  constexpr int CH = sizeof(MT) == 2 ? 1 : 4;
  constexpr int NW = AccIO<CH>::NW;
  // accumulator headroom: every limb sum must stay below 2^64 over the whole
  // reduction dimension (entries < 2^16 per product chunk, 2 products per
  // accumulator for int64)
  const uint64_t klen = transpose ? rows : cols;
  if (klen > (CH == 1 ? (1u << 16) : (1u << 15))) return kErrUnsupported;
  // warps wanted (ZKL_MV_WARPS overrides, for tuning)
  static const uint64_t kWarps = [] {
    const char* e = getenv("ZKL_MV_WARPS");
    return e ? (uint64_t)atoi(e) : (uint64_t)(24 * kSMs);
  }();
  uint64_t nchunks, nout;
  void* ws;
  int rc;
  if (!transpose && CH == 1) {
    // warp-per-row-group kernel (lanes along columns); ZKL_MVW_RW (2 / 4 rows
    // per warp) and ZKL_MVW_WAVES (target blocks per SM) are tuning overrides
    static const int kRw = [] {
      const char* e = getenv("ZKL_MVW_RW");
      return e && atoi(e) == 4 ? 4 : 2;
    }();
    static const uint64_t kWaves = [] {
      const char* e = getenv("ZKL_MVW_WAVES");
      return e ? (uint64_t)atoi(e) : (uint64_t)2;
    }();
    static const bool kTc = [] {
      const char* e = getenv("ZKL_MV_TC");
      return !(e && atoi(e) == 0);
    }();
    if (kTc && rows % 16 == 0 && cols % 32 == 0) {
      nchunks = (cols + kTcK - 1) / kTcK;
      nout = rows;
      rc = scratch_reserve(rows * NW * 8 + 128, &ws, s);
      if (rc) return rc;
      ZKL_CUDA(cudaMemsetAsync(ws, 0, rows * NW * 8 + 64, s));
      const size_t smem = 32 * (kTcK + 32);
      static bool tc_attr = false;
      if (!tc_attr) {
        ZKL_CUDA(cudaFuncSetAttribute(k_mvt_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        tc_attr = true;
      }
      dim3 g((unsigned)((rows + 127) / 128), (unsigned)nchunks);
      k_mvt_rows<<<g, 256, smem, s>>>((const int16_t*)M, rows, cols, x, (uint64_t*)ws);
      ZKL_LAUNCH_CHECK();
      goto finish;
    }
    const int RW = kRw;
    if (cols % 128) return kErrUnsupported;
    const uint64_t rblocks = (rows + 8 * RW - 1) / (8 * RW);
    uint64_t cs = (kWaves * (uint64_t)kSMs + rblocks - 1) / rblocks;  // >= kWaves blocks per SM
    const uint64_t max_cs = cols / 512;  // >= 512 columns per chunk
    if (cs > max_cs) cs = max_cs;
    if (cs < 1) cs = 1;
    uint64_t cch = (cols + cs - 1) / cs;
    cch = (cch + 127) / 128 * 128;
    if (cch > 2048) {  // the x staging holds at most 8 elements per thread
      cch = 2048;
    }
    static const uint64_t kGroups = [] {  // row groups per warp (grid-stride)
      const char* e = getenv("ZKL_MVW_GROUPS");
      return e ? (uint64_t)atoi(e) : (uint64_t)1;
    }();
    nchunks = (cols + cch - 1) / cch;
    nout = rows;
    rc = scratch_reserve(rows * NW * 8 + 128, &ws, s);
    if (rc) return rc;
    ZKL_CUDA(cudaMemsetAsync(ws, 0, rows * NW * 8 + 64, s));
    const size_t smem = cch * 32;
    static bool attr = false;
    if (!attr) {
      ZKL_CUDA(cudaFuncSetAttribute(k_mvw_rows<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    160 * 1024));
      ZKL_CUDA(cudaFuncSetAttribute(k_mvw_rows<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    160 * 1024));
      attr = true;
    }
    dim3 g((unsigned)((rblocks + kGroups - 1) / kGroups), (unsigned)nchunks);
    if (RW == 2)
      k_mvw_rows<2><<<g, 256, smem, s>>>((const int16_t*)M, rows, cols, x, cch, (uint64_t*)ws);
    else
      k_mvw_rows<4><<<g, 256, smem, s>>>((const int16_t*)M, rows, cols, x, cch, (uint64_t*)ws);
    ZKL_LAUNCH_CHECK();
  } else if (!transpose) {
    constexpr int R = 1;
    if (cols % 32) return kErrUnsupported;
    const uint64_t threads = (rows + R - 1) / R;
    uint64_t cs = (kWarps * 32 + threads - 1) / threads;
    const uint64_t max_cs = (cols + 63) / 64;  // >= 64 columns per chunk
    if (cs > max_cs) cs = max_cs;
    if (cs < 1) cs = 1;
    uint64_t cch = (cols + cs - 1) / cs;
    cch = (cch + 31) / 32 * 32;  // keep 64-byte steps aligned
    if (cch * sizeof(fr_t) > 96 * 1024) return kErrUnsupported;
    nchunks = (cols + cch - 1) / cch;
    nout = rows;
    rc = scratch_reserve(rows * NW * 8 + 128, &ws, s);
    if (rc) return rc;
    ZKL_CUDA(cudaMemsetAsync(ws, 0, rows * NW * 8 + 64, s));
    dim3 g((unsigned)((threads + 255) / 256), (unsigned)nchunks);
    const size_t smem = cch * sizeof(fr_t);
    if (smem > 48 * 1024)
      ZKL_CUDA(cudaFuncSetAttribute(k_mvf_rows<MT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    k_mvf_rows<MT, R><<<g, 256, smem, s>>>(M, rows, cols, x, cch, (uint64_t*)ws);
    ZKL_LAUNCH_CHECK();
  } else {
    static const bool kTcCols = [] {
      const char* e = getenv("ZKL_MV_TC");
      return !(e && atoi(e) == 0);
    }();
    if (CH == 1 && kTcCols && cols % 16 == 0) {
      nchunks = (rows + kTcR - 1) / kTcR;
      if (nchunks > 65535) return kErrUnsupported;
      nout = cols;
      rc = scratch_reserve(cols * NW * 8 + 128, &ws, s);
      if (rc) return rc;
      ZKL_CUDA(cudaMemsetAsync(ws, 0, cols * NW * 8 + 64, s));
      const size_t smem = kTcR * kTcMP + 32 * (kTcR + 16);
      static bool tcc_attr = false;
      if (!tcc_attr) {
        ZKL_CUDA(cudaFuncSetAttribute(k_mvt_cols, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        tcc_attr = true;
      }
      dim3 g((unsigned)((cols + kTcC - 1) / kTcC), (unsigned)nchunks);
      k_mvt_cols<<<g, 256, smem, s>>>((const int16_t*)M, rows, cols, x, (uint64_t*)ws);
      ZKL_LAUNCH_CHECK();
      goto finish;
    }
    constexpr int V = sizeof(MT) == 2 ? 2 : 1;
    if (cols % V) return kErrUnsupported;
    const uint64_t threads = cols / V;
    uint64_t rs = (kWarps * 32 + threads - 1) / threads;
    const uint64_t max_rs = (rows + 31) / 32;  // >= 32 rows per chunk
    if (rs > max_rs) rs = max_rs;
    if (rs < 1) rs = 1;
    uint64_t rch = (rows + rs - 1) / rs;
    if (rch * sizeof(fr_t) > 96 * 1024) return kErrUnsupported;
    nchunks = (rows + rch - 1) / rch;
    if (nchunks > 65535) return kErrUnsupported;
    nout = cols;
    rc = scratch_reserve(cols * NW * 8 + 128, &ws, s);
    if (rc) return rc;
    ZKL_CUDA(cudaMemsetAsync(ws, 0, cols * NW * 8 + 64, s));
    dim3 g((unsigned)((threads + 255) / 256), (unsigned)nchunks);
    const size_t smem = rch * sizeof(fr_t);
    if (smem > 48 * 1024)
      ZKL_CUDA(cudaFuncSetAttribute(k_mvf_cols<MT, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    k_mvf_cols<MT, V><<<g, 256, smem, s>>>(M, rows, cols, x, rch, (uint64_t*)ws);
    ZKL_LAUNCH_CHECK();
  }
finish:
  // y = reduce(acc) - OFF * sum(x); OFF (2^15 or 2^63) in Montgomery form
  static fr_t offr = [] {
    fr_t v = Fr255::zero();
    if (CH == 1) v.v[0] = 1u << 15;
    else v.v[1] = 1u << 31;
    return Fr255::to_mont(v);
  }();
  const uint64_t* sumx = (const uint64_t*)ws + nout * NW;
  k_mvf_finish<CH><<<(unsigned)((nout + 255) / 256), 256, 0, s>>>((const uint64_t*)ws, nout, sumx,
                                                                   offr, y);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

template <class F, class MT>
static int matvec_impl(const void* Mv, uint64_t rows, uint64_t cols, int transpose,
                       const void* xv, void* yv, cudaStream_t s) {
  using T = typename F::T;
  const MT* M = (const MT*)Mv;
  const T* x = (const T*)xv;
  T* y = (T*)yv;
  constexpr int kWant = 4 * kSMs;  // blocks to aim for
  constexpr size_t kSmemCap = 40 * 1024;
  const size_t per_x = sizeof(T) * (Mac<F, MT>::kSigned ? 2 : 1);
  uint64_t nchunks, nout = transpose ? cols : rows;
  void* ws;
  int rc;
  if (!transpose) {
    constexpr int VEC = (sizeof(MT) >= 16) ? 1 : (int)(16 / sizeof(MT));
    const bool aligned = ((uintptr_t)M % 16 == 0) && (cols % VEC == 0);
    const uint64_t rb = (rows + 255) / 256;
    uint64_t cs = (kWant + rb - 1) / rb;
    const uint64_t max_cs = (cols + 63) / 64;
    if (cs > max_cs) cs = max_cs;
    if (cs < 1) cs = 1;
    uint64_t cch = (cols + cs - 1) / cs;
    const uint64_t cap = kSmemCap / per_x;
    if (cch > cap) cch = cap;
    cch = (cch + 7) / 8 * 8;
    nchunks = (cols + cch - 1) / cch;
    rc = scratch_reserve(nchunks * rows * sizeof(T), &ws, s);
    if (rc) return rc;
    const size_t smem = cch * per_x;
    dim3 g((unsigned)rb, (unsigned)nchunks);
    if (aligned && VEC > 1)
      k_mv_rows<F, MT, VEC><<<g, 256, smem, s>>>(M, rows, cols, x, cch, (T*)ws);
    else
      k_mv_rows<F, MT, 1><<<g, 256, smem, s>>>(M, rows, cols, x, cch, (T*)ws);
    ZKL_LAUNCH_CHECK();
  } else {
    int cw = 1;
    while (cw < 256 && (uint64_t)cw < cols) cw <<= 1;
    const uint64_t cb = (cols + cw - 1) / cw;
    const uint64_t ngrp = 256 / cw;
    uint64_t rs = (kWant + cb - 1) / cb;
    const uint64_t max_rs = (rows + ngrp * 4 - 1) / (ngrp * 4);
    if (rs > max_rs) rs = max_rs;
    if (rs < 1) rs = 1;
    uint64_t rch = (rows + rs - 1) / rs;
    const uint64_t cap = (kSmemCap - 256 * sizeof(T)) / per_x;
    if (rch > cap) rch = cap;
    nchunks = (rows + rch - 1) / rch;
    if (nchunks > 65535) { set_error("matvec: too many row chunks"); return kErrArg; }
    rc = scratch_reserve(nchunks * cols * sizeof(T), &ws, s);
    if (rc) return rc;
    const size_t smem = rch * per_x + 256 * sizeof(T);
    dim3 g((unsigned)cb, (unsigned)nchunks);
    k_mv_cols<F, MT><<<g, 256, smem, s>>>(M, rows, cols, x, cw, rch, (T*)ws);
    ZKL_LAUNCH_CHECK();
  }
  k_mv_reduce<F><<<grid_for(nout * 32, 256, 8), 256, 0, s>>>((const T*)ws, nchunks, nout, y);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

// mad.wide kernels: default for int16 matrices (faster on B200); int64 stays
// on the wide-accumulator kernels unless ZKL_MATVEC_FAST64 is set (the
// 4-chunk mad.wide form measured slower).  ZKL_MATVEC_SLOW=1 disables them.
static bool fast_enabled() {
  static const bool on = getenv("ZKL_MATVEC_SLOW") == nullptr;
  return on;
}

template <class F>
int op_matvec(int mtype, const void* M, uint64_t rows, uint64_t cols, int transpose,
              const void* x, void* y, cudaStream_t s) {
  if (!rows || !cols) { set_error("matvec: empty matrix"); return kErrArg; }
  switch (mtype) {
    case 0: return matvec_impl<F, typename F::T>(M, rows, cols, transpose, x, y, s);
    case 1:
      if constexpr (F::kId == 0) {
        if (fast_enabled()) {
          int rc = matvec_fast<int16_t>((const int16_t*)M, rows, cols, transpose,
                                        (const fr_t*)x, (fr_t*)y, s);
          if (rc != kErrUnsupported) return rc;
        }
      }
      return matvec_impl<F, int16_t>(M, rows, cols, transpose, x, y, s);
    case 2: return matvec_impl<F, int32_t>(M, rows, cols, transpose, x, y, s);
    case 3:
      if constexpr (F::kId == 0) {
        if (fast_enabled() && t64_enabled()) {
          int rc = matvec_t64((const int64_t*)M, rows, cols, transpose, (const fr_t*)x, (fr_t*)y,
                              s);
          if (rc != kErrUnsupported) return rc;
        }
        if (fast_enabled() && getenv("ZKL_MATVEC_FAST64")) {
          int rc = matvec_fast<int64_t>((const int64_t*)M, rows, cols, transpose,
                                        (const fr_t*)x, (fr_t*)y, s);
          if (rc != kErrUnsupported) return rc;
        }
      }
      return matvec_impl<F, int64_t>(M, rows, cols, transpose, x, y, s);
  }
  set_error("matvec: bad matrix type %d", mtype);
  return kErrArg;
}

template int op_matvec<Fr255>(int, const void*, uint64_t, uint64_t, int, const void*, void*,
                              cudaStream_t);
template int op_matvec<M61>(int, const void*, uint64_t, uint64_t, int, const void*, void*,
                            cudaStream_t);

}  // namespace zkl
