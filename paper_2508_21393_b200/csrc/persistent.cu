// Persistent whole-sumcheck engine (sumcheck.py:108-130 after _absorb_claim).
//
// ONE cooperative launch runs every round of a claim.  Per round j:
//   1. every thread folds its pairs by r_{j-1} (in place) and accumulates
//      shape-specific raw sums (sumcheck.py:110-123 / 129);
//   2. warp shuffles + shared memory reduce them as WIDE integers (9 x 32-bit
//      words for Fr: no modular reduction on the reduction tree);
//   3. each block stores its partial, fences, and takes a ticket; the LAST
//      block sums the partials and writes them to a mailbox in mapped pinned
//      host memory as tagged 64-bit words (payload | round seq << 32);
//   4. the host reduces mod p, finishes the evaluations (term coefficients,
//      post scalars, the quadratic-product identities), appends them to the
//      native SHAKE-256 transcript, squeezes r_j and writes it back as tagged
//      words; the "drawn" state update (2 Keccak-f) runs after the write, off
//      the critical path;
//   5. each block polls the tagged challenge (directly over PCIe for small
//      grids, else block 0 relays it through an L2 slot).
// No kernel launches, copies, stream syncs or grid barriers per round.  The
// host's challenge publication orders every block's table writes of round j
// before any read of round j+1 (the last block saw all tickets before
// publishing; tables are read with ld.cg, bypassing L1).
//
// Shapes (detected from the term list on the host):
//   GENERIC  : any terms; device applies coefficients (combine, sumcheck.py:70)
//   PROD2    : c * t_a t_b              -- zkMat U/W phases; 3 mults per pair
//   PROD3    : c * t_a t_b t_c          -- elementprod; 7 mults per pair
//   SUM2PROD2: c0 t_a t_b + c1 t_a t_c  -- zkMat V phase; 6 mults per pair
// For the quadratic shapes the device returns (sum f0 g0, sum f1 g1,
// sum fd gd) and the host forms p(2) = 2p(1) - p(0) + 2c, p(3) = 3p(1) - 2p(0)
// + 6c -- exact identities of the same polynomial, computed from the tables,
// never derived from the claimed sum (hard part 3).
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <vector>

#include "hostfield.h"
#include "phase.cuh"
#include "round_eval.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace zkl {

// ---------------------------------------------------------------------------
// wide (unreduced) sums for the reduction tree
template <class F>
struct Red;

template <>
struct Red<Fr255> {
  static constexpr int NW = 9;
  struct W {
    uint32_t w[9];
  };
  ZKL_D static W from(const fr_t& x) {
    W r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.w[i] = x.v[i];
    r.w[8] = 0;
    return r;
  }
  ZKL_D static W zero() {
    W r;
#pragma unroll
    for (int i = 0; i < 9; i++) r.w[i] = 0;
    return r;
  }
  ZKL_D static W add(const W& a, const W& b) {
    W s;
    asm("add.cc.u32  %0, %9, %18;\n\t"
        "addc.cc.u32 %1, %10, %19;\n\t"
        "addc.cc.u32 %2, %11, %20;\n\t"
        "addc.cc.u32 %3, %12, %21;\n\t"
        "addc.cc.u32 %4, %13, %22;\n\t"
        "addc.cc.u32 %5, %14, %23;\n\t"
        "addc.cc.u32 %6, %15, %24;\n\t"
        "addc.cc.u32 %7, %16, %25;\n\t"
        "addc.u32    %8, %17, %26;\n\t"
        : "=r"(s.w[0]), "=r"(s.w[1]), "=r"(s.w[2]), "=r"(s.w[3]), "=r"(s.w[4]), "=r"(s.w[5]),
          "=r"(s.w[6]), "=r"(s.w[7]), "=r"(s.w[8])
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(a.w[4]), "r"(a.w[5]),
          "r"(a.w[6]), "r"(a.w[7]), "r"(a.w[8]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]),
          "r"(b.w[3]), "r"(b.w[4]), "r"(b.w[5]), "r"(b.w[6]), "r"(b.w[7]), "r"(b.w[8]));
    return s;
  }
  ZKL_D static W shfl_down(const W& a, int off) {
    W r;
#pragma unroll
    for (int i = 0; i < 9; i++) r.w[i] = __shfl_down_sync(kFull, a.w[i], off);
    return r;
  }
  ZKL_D static W shfl_xor(const W& a, int off) {
    W r;
#pragma unroll
    for (int i = 0; i < 9; i++) r.w[i] = __shfl_xor_sync(kFull, a.w[i], off);
    return r;
  }
  ZKL_D static uint32_t word(const W& a, int i) { return a.w[i]; }
};

template <>
struct Red<M61> {
  static constexpr int NW = 4;
  struct W {
    uint64_t lo, hi;
  };
  ZKL_D static W from(uint64_t x) { return W{x, 0}; }
  ZKL_D static W zero() { return W{0, 0}; }
  ZKL_D static W add(const W& a, const W& b) {
    W s;
    s.lo = a.lo + b.lo;
    s.hi = a.hi + b.hi + (s.lo < a.lo ? 1 : 0);
    return s;
  }
  ZKL_D static W shfl_down(const W& a, int off) {
    return W{__shfl_down_sync(kFull, a.lo, off), __shfl_down_sync(kFull, a.hi, off)};
  }
  ZKL_D static W shfl_xor(const W& a, int off) {
    return W{__shfl_xor_sync(kFull, a.lo, off), __shfl_xor_sync(kFull, a.hi, off)};
  }
  ZKL_D static uint32_t word(const W& a, int i) {
    const uint64_t v = i < 2 ? a.lo : a.hi;
    return (uint32_t)(v >> (32 * (i & 1)));
  }
};

// ---------------------------------------------------------------------------
// Lane mode (small rounds).  A round whose pairs fit in one pass is a pure
// latency problem, and one thread doing all of a pair's products serialises
// them (the carry chains of independent Montgomery products do not overlap
// well).  Instead a group of L lanes owns a pair: lane q < 2k folds table
// q/2, half q%2 (one product), the folded values are exchanged with
// shuffles, and each lane computes one output product.  Critical path: one
// fold product + one (PROD2, SUM2PROD2) or two (PROD3) evaluation products.
inline int lanes_for(int shape, int k) {
  if (shape == kGeneric || shape == kLogupTiled) return 0;
  const int nout = shape == kProd2 ? 3 : shape == kProd3 ? 4 : shape == kLogup ? 16
                 : shape == kZkMat ? 7 : 6;
  const int need = 2 * k > nout ? 2 * k : nout;  // fold lanes / output lanes
  return need <= 4 ? 4 : need <= 8 ? 8 : 16;
}

template <class F>
ZKL_D typename F::T shfl_elem(const typename F::T& x, int src) {
  return shfl_idx(x, src);
}

template <class F, int MAXK>
ZKL_D typename F::T lane_fold(const TablePtrs<F, MAXK>& tabs, int k, uint64_t i, uint64_t half,
                              bool fold, const typename F::T& r, int q, bool active) {
  using T = typename F::T;
  T v = F::zero();
  if (active && q < 2 * k) {
    T* t = tabs.t[q >> 1];
    const uint64_t m = i + (uint64_t)(q & 1) * half;
    if (fold) {
      const T a = ld_cg(t + m), b = ld_cg(t + m + 2 * half);
      v = F::add(a, F::mul(r, F::sub(b, a)));
      t[m] = v;
    } else {
      v = ld_cg(t + m);
    }
  }
  return v;
}

// x in {lo, hi, hi - lo} by selector s in {0, 1, 2}
template <class F>
ZKL_D typename F::T pick3(const typename F::T& lo, const typename F::T& hi, int s) {
  return s == 0 ? lo : (s == 1 ? hi : F::sub(hi, lo));
}

// ---------------------------------------------------------------------------
// evaluators: pair() accumulates NA field sums, finish() -> NOUT raw outputs
// minimum resident blocks per SM for the grid kernel of the dense
// evaluators (__launch_bounds__): 1 lets ptxas use 255 registers per thread
// (8 warps / SM), 2 caps it at 128 (16 warps / SM, more latency hiding for
// the Montgomery chains, some spilling); measured in DESIGN.md sec. 4e
#ifndef ZKL_DENSE_MINB
#define ZKL_DENSE_MINB 1
#endif
template <class F, int MAXK>
struct EvGeneric {
  using T = typename F::T;
  static constexpr int kMinBlocks = ZKL_DENSE_MINB;
  static constexpr bool kGeneric = true;
  static constexpr int NA = 4, NOUT = 4;
  ZKL_D static void pair(T (&cur)[MAXK], const T (&df)[MAXK], int k, const Terms<F>& tm,
                         T (&acc)[NA]) {
    acc[0] = F::add(acc[0], combine_terms<F, MAXK>(cur, tm));
#pragma unroll
    for (int x = 1; x < 4; x++) {
      if (x <= tm.degree) {
#pragma unroll
        for (int j = 0; j < MAXK; j++)
          if (j < k) cur[j] = F::add(cur[j], df[j]);
        acc[x] = F::add(acc[x], combine_terms<F, MAXK>(cur, tm));
      }
    }
  }
  ZKL_D static void finish(const T (&acc)[NA], T (&out)[NOUT]) {
#pragma unroll
    for (int x = 0; x < 4; x++) out[x] = acc[x];
  }
  ZKL_D static T lane(const T&, int, int, bool, const Terms<F>&) { return F::zero(); }
};

template <class F, int MAXK>
struct EvProd2 {
  using T = typename F::T;
  static constexpr int kMinBlocks = ZKL_DENSE_MINB;
  static constexpr bool kGeneric = false;
  static constexpr int NA = 3, NOUT = 3;
  ZKL_D static void pair(T (&cur)[MAXK], const T (&df)[MAXK], int, const Terms<F>& tm,
                         T (&acc)[NA]) {
    const int a = tm.fi[0][0], b = tm.fi[0][1];
    const T f0 = select_tab<F, MAXK>(cur, a), fd = select_tab<F, MAXK>(df, a);
    const T g0 = select_tab<F, MAXK>(cur, b), gd = select_tab<F, MAXK>(df, b);
    T p0, p1, pc;
    F::mul3(f0, g0, F::add(f0, fd), F::add(g0, gd), fd, gd, p0, p1, pc);
    acc[0] = F::add(acc[0], p0);
    acc[1] = F::add(acc[1], p1);
    acc[2] = F::add(acc[2], pc);
  }
  ZKL_D static void finish(const T (&acc)[NA], T (&out)[NOUT]) {
#pragma unroll
    for (int q = 0; q < 3; q++) out[q] = acc[q];
  }
  // lane mode: output q = [f0 g0, f1 g1, fd gd][q]
  ZKL_D static T lane(const T& v, int q, int gb, bool active, const Terms<F>& tm) {
    const int a = tm.fi[0][0], b = tm.fi[0][1];
    const T fl = shfl_elem<F>(v, gb + 2 * a), fh = shfl_elem<F>(v, gb + 2 * a + 1);
    const T gl = shfl_elem<F>(v, gb + 2 * b), gh = shfl_elem<F>(v, gb + 2 * b + 1);
    const int s = q < 3 ? q : 0;
    const T p = F::mul(pick3<F>(fl, fh, s), pick3<F>(gl, gh, s));
    return (active && q < 3) ? p : F::zero();
  }
};

template <class F, int MAXK>
struct EvSum2Prod2 {
  using T = typename F::T;
  static constexpr int kMinBlocks = ZKL_DENSE_MINB;
  static constexpr bool kGeneric = false;
  static constexpr int NA = 6, NOUT = 6;
  ZKL_D static void pair(T (&cur)[MAXK], const T (&df)[MAXK], int, const Terms<F>& tm,
                         T (&acc)[NA]) {
    const int a = tm.fi[0][0], b = tm.fi[0][1], c = tm.fi[1][1];
    const T f0 = select_tab<F, MAXK>(cur, a), fd = select_tab<F, MAXK>(df, a);
    const T g0 = select_tab<F, MAXK>(cur, b), gd = select_tab<F, MAXK>(df, b);
    const T h0 = select_tab<F, MAXK>(cur, c), hd = select_tab<F, MAXK>(df, c);
    const T f1 = F::add(f0, fd);
    T m[6];
    F::mul4(f0, g0, f0, h0, f1, F::add(g0, gd), f1, F::add(h0, hd), m[0], m[3], m[1], m[4]);
    F::mul2(fd, gd, fd, hd, m[2], m[5]);
#pragma unroll
    for (int q = 0; q < 6; q++) acc[q] = F::add(acc[q], m[q]);
  }
  ZKL_D static void finish(const T (&acc)[NA], T (&out)[NOUT]) {
#pragma unroll
    for (int q = 0; q < 6; q++) out[q] = acc[q];
  }
  // lane mode: output q = [f0 g0, f1 g1, fd gd, f0 h0, f1 h1, fd hd][q]
  ZKL_D static T lane(const T& v, int q, int gb, bool active, const Terms<F>& tm) {
    const int a = tm.fi[0][0], y = q < 3 ? tm.fi[0][1] : tm.fi[1][1];
    const T fl = shfl_elem<F>(v, gb + 2 * a), fh = shfl_elem<F>(v, gb + 2 * a + 1);
    const T yl = shfl_elem<F>(v, gb + 2 * y), yh = shfl_elem<F>(v, gb + 2 * y + 1);
    const int s = q < 6 ? q % 3 : 0;
    const T p = F::mul(pick3<F>(fl, fh, s), pick3<F>(yl, yh, s));
    return (active && q < 6) ? p : F::zero();
  }
};

// quadratic-product helper: (c0, c1, c2) -> p(0..3)
template <class F>
ZKL_D void quad_evals(const typename F::T& c0, const typename F::T& c1, const typename F::T& c2,
                      typename F::T* out) {
  using T = typename F::T;
  const T two_c1 = F::add(c1, c1), two_c2 = F::add(c2, c2);
  out[0] = c0;
  out[1] = c1;
  out[2] = F::sub(F::add(two_c1, two_c2), c0);                          // 2c1 - c0 + 2c2
  const T six_c2 = F::add(F::add(two_c2, two_c2), two_c2);
  out[3] = F::sub(F::add(F::add(two_c1, c1), six_c2), F::add(c0, c0));  // 3c1 - 2c0 + 6c2
}

template <class F, int MAXK>
struct EvProd3 {
  using T = typename F::T;
  static constexpr int kMinBlocks = ZKL_DENSE_MINB;
  static constexpr bool kGeneric = false;
  static constexpr int NA = 4, NOUT = 4;
  ZKL_D static void pair(T (&cur)[MAXK], const T (&df)[MAXK], int, const Terms<F>& tm,
                         T (&acc)[NA]) {
    const int a = tm.fi[0][0], b = tm.fi[0][1], c = tm.fi[0][2];
    const T e0 = select_tab<F, MAXK>(cur, a), ed = select_tab<F, MAXK>(df, a);
    const T a0 = select_tab<F, MAXK>(cur, b), ad = select_tab<F, MAXK>(df, b);
    const T b0 = select_tab<F, MAXK>(cur, c), bd = select_tab<F, MAXK>(df, c);
    T q[4], q0, q1, qc;
    F::mul3(e0, a0, F::add(e0, ed), F::add(a0, ad), ed, ad, q0, q1, qc);
    quad_evals<F>(q0, q1, qc, q);
    const T b1 = F::add(b0, bd), b2 = F::add(b1, bd), b3 = F::add(b2, bd);
    T m[4];
    F::mul4(q[0], b0, q[1], b1, q[2], b2, q[3], b3, m[0], m[1], m[2], m[3]);
#pragma unroll
    for (int x = 0; x < 4; x++) acc[x] = F::add(acc[x], m[x]);
  }
  ZKL_D static void finish(const T (&acc)[NA], T (&out)[NOUT]) {
#pragma unroll
    for (int x = 0; x < 4; x++) out[x] = acc[x];
  }
  // lane mode: level 1 q(x) = e(x) a(x) from 3 lanes, level 2 output x =
  // q(x) b(x) for x = 0..3
  ZKL_D static T lane(const T& v, int q, int gb, bool active, const Terms<F>& tm) {
    const int ie = tm.fi[0][0], ia = tm.fi[0][1], ib = tm.fi[0][2];
    const T el = shfl_elem<F>(v, gb + 2 * ie), eh = shfl_elem<F>(v, gb + 2 * ie + 1);
    const T al = shfl_elem<F>(v, gb + 2 * ia), ah = shfl_elem<F>(v, gb + 2 * ia + 1);
    const int s = q < 3 ? q : 0;
    const T p1 = F::mul(pick3<F>(el, eh, s), pick3<F>(al, ah, s));
    const T q0 = shfl_elem<F>(p1, gb), q1 = shfl_elem<F>(p1, gb + 1);
    const T qc = shfl_elem<F>(p1, gb + 2);
    T qx[4];
    quad_evals<F>(q0, q1, qc, qx);
    const T bl = shfl_elem<F>(v, gb + 2 * ib), bh = shfl_elem<F>(v, gb + 2 * ib + 1);
    const T bd = F::sub(bh, bl);
    const int x = q & 3;
    T bx = x == 0 ? bl : bh;
    if (x >= 2) bx = F::add(bx, bd);
    if (x == 3) bx = F::add(bx, bd);
    T qq = qx[0];
    if (x == 1) qq = qx[1];
    if (x == 2) qq = qx[2];
    if (x == 3) qq = qx[3];
    const T m = F::mul(qq, bx);
    return (active && q < 4) ? m : F::zero();
  }
};

// The reference's replicated zkMat claim (gadgets.py:241-251): terms
//   c0 E A B + c1 E C   (E shared).
// Raw sums: [0..3] sum E(x) A(x) B(x), x = 0..3 (as PROD3: 7 products);
// [4..6] E C as (lo lo, hi hi, slope slope) (3 products).  10 products per
// pair instead of the generic term loop.
template <class F, int MAXK>
struct EvZkMat {
  using T = typename F::T;
  static constexpr int kMinBlocks = ZKL_DENSE_MINB;
  static constexpr bool kGeneric = false;
  static constexpr int NA = 7, NOUT = 7;
  ZKL_D static void pair(T (&cur)[MAXK], const T (&df)[MAXK], int, const Terms<F>& tm,
                         T (&acc)[NA]) {
    const int ie = tm.fi[0][0], ia = tm.fi[0][1], ib = tm.fi[0][2], ic = tm.fi[1][1];
    const T e0 = select_tab<F, MAXK>(cur, ie), ed = select_tab<F, MAXK>(df, ie);
    const T a0 = select_tab<F, MAXK>(cur, ia), ad = select_tab<F, MAXK>(df, ia);
    const T b0 = select_tab<F, MAXK>(cur, ib), bd = select_tab<F, MAXK>(df, ib);
    const T c0 = select_tab<F, MAXK>(cur, ic), cd = select_tab<F, MAXK>(df, ic);
    const T e1 = F::add(e0, ed);
    T q[4], q0, q1, qc, m4, m5;
    F::mul4(e0, a0, e1, F::add(a0, ad), ed, ad, e0, c0, q0, q1, qc, m4);
    quad_evals<F>(q0, q1, qc, q);
    const T b1 = F::add(b0, bd), b2 = F::add(b1, bd), b3 = F::add(b2, bd);
    T m[4];
    F::mul4(q[0], b0, q[1], b1, q[2], b2, q[3], b3, m[0], m[1], m[2], m[3]);
    T m6;
    F::mul2(e1, F::add(c0, cd), ed, cd, m5, m6);
#pragma unroll
    for (int x = 0; x < 4; x++) acc[x] = F::add(acc[x], m[x]);
    acc[4] = F::add(acc[4], m4);
    acc[5] = F::add(acc[5], m5);
    acc[6] = F::add(acc[6], m6);
  }
  ZKL_D static void finish(const T (&acc)[NA], T (&out)[NOUT]) {
#pragma unroll
    for (int x = 0; x < NOUT; x++) out[x] = acc[x];
  }
  // lane mode: lanes 0..3 are PROD3's two levels (q(x) = e(x) a(x), then
  // q(x) b(x)); lanes 4..6 compute e c at (lo, hi, slope) in the second level
  ZKL_D static T lane(const T& v, int q, int gb, bool active, const Terms<F>& tm) {
    const int ie = tm.fi[0][0], ia = tm.fi[0][1], ib = tm.fi[0][2], ic = tm.fi[1][1];
    const T el = shfl_elem<F>(v, gb + 2 * ie), eh = shfl_elem<F>(v, gb + 2 * ie + 1);
    const T al = shfl_elem<F>(v, gb + 2 * ia), ah = shfl_elem<F>(v, gb + 2 * ia + 1);
    const int s = q < 3 ? q : 0;
    const T p1 = F::mul(pick3<F>(el, eh, s), pick3<F>(al, ah, s));
    const T q0 = shfl_elem<F>(p1, gb), q1 = shfl_elem<F>(p1, gb + 1);
    const T qc = shfl_elem<F>(p1, gb + 2);
    T qx[4];
    quad_evals<F>(q0, q1, qc, qx);
    const T bl = shfl_elem<F>(v, gb + 2 * ib), bh = shfl_elem<F>(v, gb + 2 * ib + 1);
    const T cl = shfl_elem<F>(v, gb + 2 * ic), ch = shfl_elem<F>(v, gb + 2 * ic + 1);
    const T bd = F::sub(bh, bl);
    const int x = q & 3;
    T bx = x == 0 ? bl : bh;
    if (x >= 2) bx = F::add(bx, bd);
    if (x == 3) bx = F::add(bx, bd);
    T qq = qx[0];
    if (x == 1) qq = qx[1];
    if (x == 2) qq = qx[2];
    if (x == 3) qq = qx[3];
    const int s2 = q >= 4 && q < 7 ? q - 4 : 0;
    const T lhs = q < 4 ? qq : pick3<F>(el, eh, s2);
    const T rhs = q < 4 ? bx : pick3<F>(cl, ch, s2);
    const T m = F::mul(lhs, rhs);
    return (active && q < 7) ? m : F::zero();
  }
};

// logUp Eq.-7 claim (lookup.py:116-126): terms
//   c0 E A S + c1 E I + c2 E B T + c3 A + c4 M B
// (E eq, A 1/(beta+s), S s+beta, I indicator, B 1/(beta+t), T t+beta, M
// multiplicities).  Raw sums returned for the host to combine with c0..c4:
//   [0..3] sum E(x) (AS)(x)      x = 0..3   (AS quadratic from 3 products)
//   [4..6] E I   as (lo lo, hi hi, slope slope)
//   [7..10] sum E(x) (BT)(x)     x = 0..3
//   [11..12] sum A lo, sum A slope (linear)
//   [13..15] M B  as (lo lo, hi hi, slope slope)
// 20 products per pair instead of ~44 for the generic term loop.
template <class F, int MAXK>
struct EvLogup {
  using T = typename F::T;
  static constexpr int kMinBlocks = ZKL_DENSE_MINB;
  static constexpr bool kGeneric = false;
  static constexpr int NA = 16, NOUT = 16;
  struct Idx {
    int e, a, s, i, b, t, m;
  };
  ZKL_D static Idx idx(const Terms<F>& tm) {
    return Idx{tm.fi[0][0], tm.fi[0][1], tm.fi[0][2], tm.fi[1][1],
               tm.fi[2][1], tm.fi[2][2], tm.fi[4][0]};
  }
  ZKL_D static void pair(T (&cur)[MAXK], const T (&df)[MAXK], int, const Terms<F>& tm,
                         T (&acc)[NA]) {
    const Idx x = idx(tm);
    const T e0 = select_tab<F, MAXK>(cur, x.e), ed = select_tab<F, MAXK>(df, x.e);
    const T a0 = select_tab<F, MAXK>(cur, x.a), ad = select_tab<F, MAXK>(df, x.a);
    const T s0 = select_tab<F, MAXK>(cur, x.s), sd = select_tab<F, MAXK>(df, x.s);
    const T i0 = select_tab<F, MAXK>(cur, x.i), id = select_tab<F, MAXK>(df, x.i);
    const T b0 = select_tab<F, MAXK>(cur, x.b), bd = select_tab<F, MAXK>(df, x.b);
    const T t0 = select_tab<F, MAXK>(cur, x.t), td = select_tab<F, MAXK>(df, x.t);
    const T m0 = select_tab<F, MAXK>(cur, x.m), md = select_tab<F, MAXK>(df, x.m);
    const T e1 = F::add(e0, ed), a1 = F::add(a0, ad), s1 = F::add(s0, sd);
    const T b1 = F::add(b0, bd), t1 = F::add(t0, td), i1 = F::add(i0, id);
    const T m1 = F::add(m0, md);
    T as[4], bt[4], p[4], q[4];
    F::mul4(a0, s0, a1, s1, ad, sd, b0, t0, p[0], p[1], p[2], q[0]);
    F::mul2(b1, t1, bd, td, q[1], q[2]);
    quad_evals<F>(p[0], p[1], p[2], as);
    quad_evals<F>(q[0], q[1], q[2], bt);
    const T e2 = F::add(e1, ed), e3 = F::add(e2, ed);
    T o[8];
    F::mul4(e0, as[0], e1, as[1], e2, as[2], e3, as[3], o[0], o[1], o[2], o[3]);
    F::mul4(e0, bt[0], e1, bt[1], e2, bt[2], e3, bt[3], o[4], o[5], o[6], o[7]);
    T ei[3], mb[3];
    F::mul3(e0, i0, e1, i1, ed, id, ei[0], ei[1], ei[2]);
    F::mul3(m0, b0, m1, b1, md, bd, mb[0], mb[1], mb[2]);
#pragma unroll
    for (int k = 0; k < 4; k++) acc[k] = F::add(acc[k], o[k]);
#pragma unroll
    for (int k = 0; k < 3; k++) acc[4 + k] = F::add(acc[4 + k], ei[k]);
#pragma unroll
    for (int k = 0; k < 4; k++) acc[7 + k] = F::add(acc[7 + k], o[4 + k]);
    acc[11] = F::add(acc[11], a0);
    acc[12] = F::add(acc[12], ad);
#pragma unroll
    for (int k = 0; k < 3; k++) acc[13 + k] = F::add(acc[13 + k], mb[k]);
  }
  ZKL_D static void finish(const T (&acc)[NA], T (&out)[NOUT]) {
#pragma unroll
    for (int q = 0; q < 16; q++) out[q] = acc[q];
  }
  // lane mode (L = 16): level-1 products on lanes 0-2 (A S), 4-6 (E I, outputs),
  // 7-9 (B T), 13-15 (M B, outputs); level-2 E(x) (AS)(x) on lanes 0-3 and
  // E(x) (BT)(x) on lanes 7-10; lanes 11/12 carry A lo / A slope.
  ZKL_D static T lane(const T& v, int q, int gb, bool active, const Terms<F>& tm) {
    const Idx x = idx(tm);
    int X = x.a, Y = x.a, sel = 0;
    if (q < 3) { X = x.a; Y = x.s; sel = q; }
    else if (q >= 4 && q < 7) { X = x.e; Y = x.i; sel = q - 4; }
    else if (q >= 7 && q < 10) { X = x.b; Y = x.t; sel = q - 7; }
    else if (q >= 13) { X = x.m; Y = x.b; sel = q - 13; }
    const T xl = shfl_elem<F>(v, gb + 2 * X), xh = shfl_elem<F>(v, gb + 2 * X + 1);
    const T yl = shfl_elem<F>(v, gb + 2 * Y), yh = shfl_elem<F>(v, gb + 2 * Y + 1);
    const T p1 = F::mul(pick3<F>(xl, xh, sel), pick3<F>(yl, yh, sel));
    const int base = q < 7 ? 0 : 7;  // which quadratic feeds level 2
    const T c0 = shfl_elem<F>(p1, gb + base), c1 = shfl_elem<F>(p1, gb + base + 1);
    const T c2 = shfl_elem<F>(p1, gb + base + 2);
    T qx[4];
    quad_evals<F>(c0, c1, c2, qx);
    const T el = shfl_elem<F>(v, gb + 2 * x.e), eh = shfl_elem<F>(v, gb + 2 * x.e + 1);
    const T ed = F::sub(eh, el);
    const int xx = (q < 4 ? q : q - 7) & 3;
    T ex = xx == 0 ? el : eh, qv = qx[0];
    if (xx >= 2) ex = F::add(ex, ed);
    if (xx == 3) ex = F::add(ex, ed);
    if (xx == 1) qv = qx[1];
    if (xx == 2) qv = qx[2];
    if (xx == 3) qv = qx[3];
    const T p2 = F::mul(ex, qv);
    const T al = shfl_elem<F>(v, gb + 2 * x.a), ah = shfl_elem<F>(v, gb + 2 * x.a + 1);
    T out;
    if (q < 4 || (q >= 7 && q < 11)) out = p2;
    else if (q == 11) out = al;
    else if (q == 12) out = F::sub(ah, al);
    else out = p1;  // 4-6 (E I) and 13-15 (M B)
    return active ? out : F::zero();
  }
};

// logUp Eq.-7 claim in its replicated form (lookup.py:188-202, secret
// larger than the table), for the rounds that bind the high log2(d/n)
// variables.  Three structural facts remove most of the work:
//  * the table side [B, T, M] depends only on the low tile_log index bits,
//    so lo == hi inside every pair: sum E B T = C_j l(x) sum_ti BT(ti)
//    eq_lo(ti) (eq tables sum to 1) and sum M B = (half / 2^tile_log)
//    sum_ti M B -- two constants the host computes once;
//  * the indicator is 1, and sum E I = C_j l(x);
//  * E is an eq table: after binding r_0..r_{j-1} it is
//    C_j * l_j(x) * eq_hi_j(k) * eq_lo(ti) for the pair (i, i + half) with
//    i = k 2^tile_log + ti, where l_j(x) = (1 - u_j) + x (2 u_j - 1) and
//    C_j = prod_{t<j} l_t(r_t).  E is never materialised or folded.
// The device sums, per round, P_c = sum_i eq_hi(k) eq_lo(ti) q_c(i) with
// q_0 = a0 s0, q_1 = a1 s1, q_2 = (a1 - a0)(s1 - s0) (A S at x = 0, 1 and
// its x^2 coefficient) plus sum a0 and sum (a1 - a0); the host builds the
// four evaluations.  Per pair: 4 products to fold A, S, 3 for q, 3 for the
// eq_hi weights (the eq_lo weight is applied once per run of one ti block).
// In round 0, when A = 1/S entrywise (tm.inv_pair), q_0 = q_1 = 1 and P_0 =
// P_1 = 1: two products per pair.
// Tables: [eq_hi (all rounds, round j's 2^(r-1-j) entries at offset
// 2^(r-1-j) - 1), A, S + beta, eq_lo (2^tile_log)].
#ifndef ZKL_TILED_MINB
#define ZKL_TILED_MINB 2
#endif
template <class F, int MAXK>
struct EvLogupTiled {
  using T = typename F::T;
  static constexpr bool kGeneric = false;
  static constexpr bool kTiled = true;
  static constexpr int kMinBlocks = ZKL_TILED_MINB;
  static constexpr int NA = 5, NOUT = 5;
  ZKL_D static void accumulate(const TablePtrs<F, MAXK>& tabs, uint64_t half, bool fold,
                               const T& r, const Terms<F>& tm, uint64_t gtid,
                               uint64_t nthreads, T (&acc)[NA]) {
    // S is kept weighted by eq_lo: S~(k, t) = eq_lo(t) S(k, t).  eq_lo depends
    // only on the low index t, which folds never touch, so S~ folds like S,
    // and a S~ = eq_lo a S puts the eq_lo weight into the q products for free.
    // Warp-steps run k-major (t inner), so the eq_hi(k) weight is applied once
    // per run of one k.  Products per pair: round 0 two (inv_pair) or five,
    // round 1 (whose fold reads the unweighted column) nine, later rounds
    // seven -- against 2 / 6 / 10 / 10 with both weights applied per pair.
    // The host un-weights the n surviving entries after the last tiled round.
    const int tl = tm.tile_log;
    const uint64_t K = half >> tl;  // pairs per low index t (a power of two)
    const int tib_log = tl - 5;
    const uint64_t steps = K << tib_log;
    const uint64_t nw = nthreads >> 5, gw = gtid >> 5;
    const uint64_t f0 = steps * gw / nw, f1 = steps * (gw + 1) / nw;
    const int lane = threadIdx.x & 31;
    const T* eh = tabs.t[0] + (K - 1);
    const T* A = tabs.t[1];
    const T* Sb = tabs.t[2];
    const T* el = tabs.t[3];
    const bool inv0 = !fold && tm.inv_pair;
    const bool first_fold = fold && (half << 2) == tm.tiled_d;  // reads the unweighted S
    const bool idx_fold = first_fold && tm.sidx != nullptr;
    T p0 = F::zero(), p1 = F::zero(), p2 = F::zero();
    uint64_t cur = ~0ull;
    auto flush = [&](uint64_t kk) {
      const T wh = eh[kk];
      if (inv0) {
        acc[2] = F::add(acc[2], F::mul(wh, p2));
      } else {
        F::mul3(wh, p0, wh, p1, wh, p2, p0, p1, p2);
        acc[0] = F::add(acc[0], p0);
        acc[1] = F::add(acc[1], p1);
        acc[2] = F::add(acc[2], p2);
      }
      p0 = p1 = p2 = F::zero();
    };
    for (uint64_t f = f0; f < f1; f++) {
      const uint64_t kk = f >> tib_log, tib = f & ((1ull << tib_log) - 1);
      if (kk != cur) {
        if (cur != ~0ull) flush(cur);
        cur = kk;
      }
      const uint64_t t = (tib << 5) | lane;
      const uint64_t i = (kk << tl) | t;
      T a0, ad, s0, s1;
      if (fold) {
        T* At = tabs.t[1];
        T* St = tabs.t[2];
        T xa, ya, xs, ys, da, db, ds, dt;
        if (idx_fold) {  // first fold: the unfolded columns are table entries
          const uint32_t j0 = __ldg(tm.sidx + i), j1 = __ldg(tm.sidx + i + half);
          const uint32_t j2 = __ldg(tm.sidx + i + 2 * half), j3 = __ldg(tm.sidx + i + 3 * half);
          xa = tm.side_a[j0];
          ya = tm.side_a[j1];
          xs = tm.side_s[j0];
          ys = tm.side_s[j1];
          da = F::sub(tm.side_a[j2], xa);
          db = F::sub(tm.side_a[j3], ya);
          ds = F::sub(tm.side_s[j2], xs);
          dt = F::sub(tm.side_s[j3], ys);
        } else {
          xa = ld_cg(At + i);
          ya = ld_cg(At + i + half);
          xs = ld_cg(St + i);
          ys = ld_cg(St + i + half);
          da = F::sub(ld_cg(At + i + 2 * half), xa);
          db = F::sub(ld_cg(At + i + 3 * half), ya);
          ds = F::sub(ld_cg(St + i + 2 * half), xs);
          dt = F::sub(ld_cg(St + i + 3 * half), ys);
        }
        F::mul4r(r, da, db, ds, dt);
        a0 = F::add(xa, da);
        const T a1 = F::add(ya, db);
        s0 = F::add(xs, ds);
        s1 = F::add(ys, dt);
        if (first_fold) {  // weight the folded S by eq_lo(t) from here on
          const T wl = el[t];
          F::mul2(wl, s0, wl, s1, s0, s1);
        }
        At[i] = a0;
        At[i + half] = a1;
        St[i] = s0;
        St[i + half] = s1;
        ad = F::sub(a1, a0);
      } else {
        T ah, sh;
        if (tm.sidx) {
          const uint32_t j0 = __ldg(tm.sidx + i), j1 = __ldg(tm.sidx + i + half);
          a0 = tm.side_a[j0];
          ah = tm.side_a[j1];
          s0 = tm.side_s[j0];
          sh = tm.side_s[j1];
        } else {
          a0 = ld_cg(A + i);
          ah = ld_cg(A + i + half);
          s0 = ld_cg(Sb + i);
          sh = ld_cg(Sb + i + half);
        }
        ad = F::sub(ah, a0);
        const T wl = el[t];
        if (inv0) {  // a S = 1 at both ends: only the slope product is needed
          acc[3] = F::add(acc[3], a0);
          acc[4] = F::add(acc[4], ad);
          const T sd = F::mul(wl, F::sub(sh, s0));
          p2 = F::add(p2, F::mul(ad, sd));
          continue;
        }
        F::mul2(wl, s0, wl, sh, s0, s1);
      }
      acc[3] = F::add(acc[3], a0);
      acc[4] = F::add(acc[4], ad);
      const T a1 = F::add(a0, ad);
      T q0, q1, q2;
      F::mul3(a0, s0, a1, s1, ad, F::sub(s1, s0), q0, q1, q2);
      p0 = F::add(p0, q0);
      p1 = F::add(p1, q1);
      p2 = F::add(p2, q2);
    }
    if (cur != ~0ull) flush(cur);
  }
  ZKL_D static void pair(T (&)[MAXK], const T (&)[MAXK], int, const Terms<F>&, T (&)[NA]) {}
  ZKL_D static void finish(const T (&acc)[NA], T (&out)[NOUT]) {
#pragma unroll
    for (int q = 0; q < NOUT; q++) out[q] = acc[q];
  }
  ZKL_D static T lane(const T&, int, int, bool, const Terms<F>&) { return F::zero(); }
};

// blocks per SM the grid kernel is compiled for (register budget): 2 for
// evaluators whose per-pair state fits 128 registers, so two blocks share an
// SM and hide the Montgomery carry-chain latency
template <class EV>
struct MinBlocks {
  template <class U>
  static constexpr int test(decltype(U::kMinBlocks)*) { return U::kMinBlocks; }
  template <class U>
  static constexpr int test(...) { return 1; }
  static constexpr int value = test<EV>(nullptr);
};

template <class EV>
struct IsTiled {
  template <class U>
  static constexpr bool test(decltype(U::kTiled)*) { return U::kTiled; }
  template <class U>
  static constexpr bool test(...) { return false; }
  static constexpr bool value = test<EV>(nullptr);
};

// Load the pair (i, i + half) of every table, folding first when FOLD:
// cur = low value, df = high - low.  All 2k fold products go through the
// 4-wide multiply (one product latency per 4 folds).
template <class F, int MAXK, bool FOLD>
ZKL_D void load_fold_pair(const TablePtrs<F, MAXK>& tabs, int k, uint64_t i, uint64_t half,
                          const typename F::T& r, typename F::T (&cur)[MAXK],
                          typename F::T (&df)[MAXK]) {
  using T = typename F::T;
  if (!FOLD) {
#pragma unroll
    for (int j = 0; j < MAXK; j++) {
      if (j < k) {
        const T* t = tabs.t[j];
        const T lo = ld_cg(t + i), hi = ld_cg(t + i + half);
        cur[j] = lo;
        df[j] = F::sub(hi, lo);
      } else {
        cur[j] = F::zero();
        df[j] = F::zero();
      }
    }
    return;
  }
  T a0[MAXK], b0[MAXK], da[MAXK], db[MAXK];
#pragma unroll
  for (int j = 0; j < MAXK; j++) {
    if (j < k) {
      const T* t = tabs.t[j];
      a0[j] = ld_cg(t + i);
      b0[j] = ld_cg(t + i + half);
      da[j] = F::sub(ld_cg(t + i + 2 * half), a0[j]);
      db[j] = F::sub(ld_cg(t + i + 3 * half), b0[j]);
    } else {
      a0[j] = b0[j] = da[j] = db[j] = F::zero();
    }
  }
#pragma unroll
  for (int j = 0; j < MAXK; j += 2) {
    if (j < k) {
      if (j + 1 < MAXK) F::mul4r(r, da[j], db[j], da[j + 1], db[j + 1]);
      else F::mul2(r, da[j], r, db[j], da[j], db[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < MAXK; j++) {
    if (j < k) {
      T* t = tabs.t[j];
      const T lo = F::add(a0[j], da[j]), hi = F::add(b0[j], db[j]);
      t[i] = lo;
      t[i + half] = hi;
      cur[j] = lo;
      df[j] = F::sub(hi, lo);
    } else {
      cur[j] = F::zero();
      df[j] = F::zero();
    }
  }
}

// ---------------------------------------------------------------------------
// tagged-word mailbox access (host-mapped memory: device reads are PCIe
// round trips, device writes are posted)
ZKL_D void st_tagged2(volatile uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
ZKL_D void ld_tagged2(const volatile uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
ZKL_D uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
ZKL_D uint64_t tag(uint32_t w, uint32_t seq) { return (uint64_t)w | ((uint64_t)seq << 32); }

constexpr uint64_t kSpinTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s
constexpr int kThreads = 256;
constexpr int kDirectPollMaxGrid = 1;

// Poll NW tagged words until all carry `seq`; payload -> out.  Returns false
// on abort / timeout.
template <int NW>
ZKL_D bool poll_tagged(const volatile uint64_t* src, uint32_t seq, uint32_t (&out)[NW],
                       const volatile uint32_t* abort_flag) {
  const uint64_t t0 = globaltimer();
  for (uint32_t spin = 1;; spin++) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < NW; i += 2) {
      uint64_t a, b = 0;
      if (i + 1 < NW) ld_tagged2(src + i, a, b);
      else a = src[i];
      ok &= (uint32_t)(a >> 32) == seq;
      out[i] = (uint32_t)a;
      if (i + 1 < NW) {
        ok &= (uint32_t)(b >> 32) == seq;
        out[i + 1] = (uint32_t)b;
      }
    }
    if (ok) return true;
    if ((spin & 63) == 0 && ((abort_flag && *abort_flag) || globaltimer() - t0 > kSpinTimeoutNs))
      return false;
  }
}

// Warp-cooperative poll: lanes < NW/2 each load one 16-byte pair of tagged
// words (independent loads, one PCIe round trip per poll; a single thread
// issuing the loads back to back pays one round trip per load).  Every lane
// of the warp must call it; on success out[0..NW) holds the payload.
// Recorded-challenge replay (ZKL_PROFILE_REPLAY, run_phase_replay): when set,
// a poll of the host challenge slot `ch` for round tag seq reads the
// pre-drawn challenge from device memory instead, so a profiler that replays
// the persistent / cluster kernels (ncu restores device memory between
// passes) sees exactly the production kernels with no host in the loop.
struct RecordedChallenges {
  const uint32_t* words;  // round j's challenge at words[j * NW] (storage form)
  const volatile uint64_t* ch;
  uint32_t seq0;
};
__device__ RecordedChallenges g_rec = {nullptr, nullptr, 0};
// replay only: blocks of the grid kernel that finished each round.  Live, the
// challenge of round j exists only after every block finished round j (the
// host draws it from the published sums), which is what orders the next
// round's reads after the other blocks' in-place folds; a recorded challenge
// is available at once, so block 0 first waits for this count.
__device__ unsigned g_rec_done = 0;

template <int NW>
ZKL_D bool warp_poll(const volatile uint64_t* src, uint32_t seq, uint32_t* out,
                     const volatile uint32_t* abort_flag) {
  const int lane = threadIdx.x & 31;
  if (g_rec.words && src == g_rec.ch) {
    if (lane < NW) out[lane] = g_rec.words[(size_t)(seq - g_rec.seq0 - 1) * NW + lane];
    __syncwarp();
    return true;
  }
  const uint64_t t0 = globaltimer();
  for (uint32_t spin = 1;; spin++) {
    uint64_t a = (uint64_t)seq << 32, b = a;
    if (lane < NW / 2) ld_tagged2(src + 2 * lane, a, b);
    const bool mine = (uint32_t)(a >> 32) == seq && (uint32_t)(b >> 32) == seq;
    if (__all_sync(kFull, mine)) {
      if (lane < NW / 2) {
        out[2 * lane] = (uint32_t)a;
        out[2 * lane + 1] = (uint32_t)b;
      }
      __syncwarp();
      return true;
    }
    if ((spin & 63) == 0) {
      int bad = lane == 0 && ((abort_flag && *abort_flag) || globaltimer() - t0 > kSpinTimeoutNs);
      if (__shfl_sync(kFull, bad, 0)) return false;
    }
  }
}

// both challenges of a paired round in one PCIe read round trip: lanes
// [0, NW/2) poll ch (tag seq), lanes [NW/2, NW) poll ch2 (tag seq + 1)
template <int NW>
ZKL_D bool warp_poll2(const volatile uint64_t* ch, const volatile uint64_t* ch2, uint32_t seq,
                      uint32_t* out, uint32_t* out2, const volatile uint32_t* abort_flag) {
  const int lane = threadIdx.x & 31;
  const bool first = lane < NW / 2;
  const int l2 = first ? lane : lane - NW / 2;
  const uint32_t want = first ? seq : seq + 1;
  const uint64_t t0 = globaltimer();
  for (uint32_t spin = 1;; spin++) {
    uint64_t a = (uint64_t)want << 32, b = a;
    if (lane < NW) ld_tagged2((first ? ch : ch2) + 2 * l2, a, b);
    const bool mine = (uint32_t)(a >> 32) == want && (uint32_t)(b >> 32) == want;
    if (__all_sync(kFull, mine)) {
      if (lane < NW) {
        uint32_t* o = first ? out : out2;
        o[2 * l2] = (uint32_t)a;
        o[2 * l2 + 1] = (uint32_t)b;
      }
      __syncwarp();
      return true;
    }
    if ((spin & 63) == 0) {
      int bad = lane == 0 && ((abort_flag && *abort_flag) || globaltimer() - t0 > kSpinTimeoutNs);
      if (__shfl_sync(kFull, bad, 0)) return false;
    }
  }
}

template <class F>
struct Words {
  static constexpr int N = F::kBytes / 4;  // 8 (Fr) or 2 (M61)
  ZKL_D static typename F::T load(const uint32_t* w) {
    typename F::T r;
    memcpy(&r, w, F::kBytes);
    return r;
  }
  ZKL_D static uint32_t word(const typename F::T& x, int i) {
    uint32_t w[N];
    memcpy(w, &x, F::kBytes);
    return w[i];
  }
};

// One round's accumulation for the calling thread: folds (if `fold`) and
// evaluates its pairs (lane mode when L > 0, else one pair per thread), then
// leaves the warp's wide sums in wsum[warp][0..NOUT).  Every thread of the
// block must call it (it ends with the warp shuffles).
// Lane mode for small rounds (L > 0), one pair per thread otherwise (large
// rounds: more independent products per thread, no shuffles; measured 45 vs
// 74 ms for the 2^25 logUp claim with lane mode forced everywhere).
template <class F, int MAXK, class EV>
ZKL_D void accumulate_round(const TablePtrs<F, MAXK>& tabs, int k, const Terms<F>& tm,
                            uint64_t half, bool fold, const typename F::T& r, int L,
                            uint64_t gtid, uint64_t nthreads,
                            typename Red<F>::W (*wsum)[EV::NOUT]) {
  using T = typename F::T;
  using R = Red<F>;
  using W = typename R::W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (!EV::kGeneric && L > 0) {
    // lane mode: groups of L lanes, one pair per group per pass
    const uint64_t ngroups = nthreads / (unsigned)L;
    const int q = lane & (L - 1), gb = lane & ~(L - 1);
    T o = F::zero();
    const uint64_t passes = (half + ngroups - 1) / ngroups;
    uint64_t i = gtid / (unsigned)L;
    for (uint64_t ps = 0; ps < passes; ps++, i += ngroups) {
      const bool active = i < half;
      const T fv = lane_fold<F, MAXK>(tabs, k, i, half, fold, r, q, active);
      o = F::add(o, EV::lane(fv, q, gb, active, tm));
    }
    W w = R::from(o);
    for (int off = 16; off >= L; off >>= 1) w = R::add(w, R::shfl_down(w, off));
    if (lane < EV::NOUT) wsum[warp][lane] = w;  // lane q < L holds output q
  } else {
    (void)L;
    T acc[EV::NA];
#pragma unroll
    for (int q = 0; q < EV::NA; q++) acc[q] = F::zero();
    if constexpr (IsTiled<EV>::value) {
      EV::accumulate(tabs, half, fold, r, tm, gtid, nthreads, acc);
    } else {
      for (uint64_t i = gtid; i < half; i += nthreads) {
        T cur[MAXK], df[MAXK];
        if (fold)
          load_fold_pair<F, MAXK, true>(tabs, k, i, half, r, cur, df);
        else
          load_fold_pair<F, MAXK, false>(tabs, k, i, half, r, cur, df);
        EV::pair(cur, df, k, tm, acc);
      }
    }
    T out[EV::NOUT];
    EV::finish(acc, out);
#pragma unroll
    for (int q = 0; q < EV::NOUT; q++) {
      W v = R::from(out[q]);
#pragma unroll
      for (int off = 16; off; off >>= 1) v = R::add(v, R::shfl_down(v, off));
      if (lane == 0) wsum[warp][q] = v;
    }
  }
}

// warp 0: sum the per-warp wide sums of the block; lane 0 gets the totals
template <class F, int NOUT>
ZKL_D void block_total(typename Red<F>::W (*wsum)[NOUT], int nwarps,
                       typename Red<F>::W (&tot)[NOUT]) {
  using R = Red<F>;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NOUT; q++) {
    typename R::W s = lane < nwarps ? wsum[lane][q] : R::zero();
#pragma unroll
    for (int off = 16; off; off >>= 1) s = R::add(s, R::shfl_down(s, off));
    tot[q] = s;
  }
}

// warp-wide: lane 0's totals -> tagged mailbox words (one 16-byte PCIe store
// per lane; a single thread issuing all of them serialises)
template <class F, int NOUT>
ZKL_D void publish_sums(const typename Red<F>::W (&tot)[NOUT], uint32_t seq, Mailbox* mb,
                        uint64_t* s_words) {
  using R = Red<F>;
  constexpr int NW = R::NW, NWORDS = NOUT * NW;
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NOUT; q++) {
#pragma unroll
      for (int w = 0; w < NW; w++) s_words[q * NW + w] = tag(R::word(tot[q], w), seq);
    }
  }
  __syncwarp();
  for (int idx = 2 * lane; idx < NWORDS; idx += 64) {
    if (idx + 1 < NWORDS)
      st_tagged2(mb->ev + idx, s_words[idx], s_words[idx + 1]);
    else
      mb->ev[idx] = s_words[idx];
  }
}

template <class F, int MAXK>
ZKL_D void publish_finals(const TablePtrs<F, MAXK>& tabs, int k, const typename F::T& r,
                          uint32_t fseq, Mailbox* mb) {
  using T = typename F::T;
  constexpr int NC = Words<F>::N;
  if (threadIdx.x < k) {
    const T* t = tabs.t[threadIdx.x];
    const T a = ld_cg(t), b = ld_cg(t + 1);
    const T f = F::add(a, F::mul(r, F::sub(b, a)));
#pragma unroll
    for (int w = 0; w < NC; w++) mb->fin[threadIdx.x * NC + w] = tag(Words<F>::word(f, w), fseq);
  }
}

// ---------------------------------------------------------------------------
// Grid kernel (large rounds): many blocks, cooperative launch for
// co-residency.  Runs rounds [j0, j1) of the claim; the LAST arriving block
// (ticket) sums the block partials and publishes; block 0 polls the
// challenge and relays it through an L2 slot.  When j1 < num_vars the
// remaining rounds continue in the cluster kernel (no finals here).
template <class F, int MAXK, class EV>
__global__ void __launch_bounds__(kThreads, MinBlocks<EV>::value)
    k_sumcheck_persistent(TablePtrs<F, MAXK> tabs, int k, int num_vars, int j0, int j1,
                          Terms<F> tm, Mailbox* mb, typename Red<F>::W* partials,
                          unsigned* ticket, uint64_t* bcast, unsigned* fail, uint32_t seq0,
                          int direct, uint64_t* trace, int L) {
  using T = typename F::T;
  using R = Red<F>;
  using W = typename R::W;
  constexpr int NC = Words<F>::N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  __shared__ W wsum[kThreads / 32][EV::NOUT];
  __shared__ T s_r;
  __shared__ int s_flag;
  __shared__ uint64_t s_words[kMbEvalWords];
  const unsigned G = gridDim.x;
  const uint64_t nthreads = (uint64_t)G * blockDim.x;
  const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  T r = F::zero();
  for (int j = j0; j < j1; j++) {
    const uint32_t seq = seq0 + (uint32_t)j + 1;
    const bool fold = j > 0;
    const bool tr0 = trace && blockIdx.x == 0 && threadIdx.x == 0;
    if (tr0) trace[j * 8 + 0] = globaltimer();
    const uint64_t tb0 = trace ? globaltimer() : 0;
    const uint64_t half = 1ull << (num_vars - 1 - j);
    // lane mode while a round needs at most (L >> 8) & 255 passes of the cluster
    const int Ll = L & 255;
    const int Lr =
        (Ll > 0 && half * (uint64_t)Ll <= nthreads * (uint64_t)((L >> 8) & 255)) ? Ll : 0;
    accumulate_round<F, MAXK, EV>(tabs, k, tm, half, fold, r, Lr, gtid, nthreads, wsum);
    if (tr0) trace[j * 8 + 1] = globaltimer();
    __syncthreads();
    if (trace && threadIdx.x == 0) {  // per-block accumulate time and SM (ZKL_TRACE)
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trace[(size_t)num_vars * 8 + ((size_t)j * G + blockIdx.x) * 2] = globaltimer() - tb0;
      trace[(size_t)num_vars * 8 + ((size_t)j * G + blockIdx.x) * 2 + 1] = smid;
    }
    if (warp == 0) {
      W v[EV::NOUT];
      block_total<F, EV::NOUT>(wsum, nwarps, v);
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < EV::NOUT; q++) partials[(size_t)blockIdx.x * EV::NOUT + q] = v[q];
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        if (g_rec.words) atomicAdd(&g_rec_done, 1u);
        s_flag = (t == G * (unsigned)(j - j0 + 1) - 1) ? 1 : 0;
        if (tr0) trace[j * 8 + 2] = globaltimer();
      }
    }
    __syncthreads();
    if (s_flag && warp == 0) {
      // last block: warp 0 sums the partials and publishes
      __threadfence();
      W tot[EV::NOUT];
#pragma unroll
      for (int q = 0; q < EV::NOUT; q++) tot[q] = R::zero();
      for (unsigned b = lane; b < G; b += 32) {
#pragma unroll
        for (int q = 0; q < EV::NOUT; q++) {
          W pv;
          const uint32_t* src =
              reinterpret_cast<const uint32_t*>(partials + (size_t)b * EV::NOUT + q);
#pragma unroll
          for (int w = 0; w < (int)(sizeof(W) / 4); w++)
            reinterpret_cast<uint32_t*>(&pv)[w] = __ldcg(src + w);
          tot[q] = R::add(tot[q], pv);
        }
      }
#pragma unroll
      for (int q = 0; q < EV::NOUT; q++) {
#pragma unroll
        for (int off = 16; off; off >>= 1) tot[q] = R::add(tot[q], R::shfl_down(tot[q], off));
      }
      if (lane == 0 && j == j1 - 1) atomicExch(ticket, 0u);  // every block has arrived
      publish_sums<F, EV::NOUT>(tot, seq, mb, s_words);
      if (trace && lane == 0) trace[j * 8 + 3] = globaltimer();
    }
    if (j == j1 - 1 && j1 < num_vars) return;  // the cluster kernel takes over
    // wait for r_j: warp 0 polls (the host mailbox directly, or block 0
    // polls it and relays through an L2 slot)
    if (warp == 0) {
      __shared__ uint32_t cw[NC];
      bool ok;
      if (direct || blockIdx.x == 0) {
        if (g_rec.words) {
          const unsigned want = G * (unsigned)(j - j0 + 1);
          while (*(volatile unsigned*)&g_rec_done < want) {
          }
        }
        ok = warp_poll<NC>(mb->ch, seq, cw, &mb->abort);
        if (!direct && ok && lane < NC)
          reinterpret_cast<volatile uint64_t*>(bcast)[lane] = tag(cw[lane], seq);
      } else {
        ok = warp_poll<NC>(bcast, seq, cw, nullptr);
      }
      if (lane == 0) {
        if (!ok) {
          *fail = 1;
          mb->status = 1;
          if (!direct && blockIdx.x == 0) {
#pragma unroll
            for (int i = 0; i < NC; i++)
              reinterpret_cast<volatile uint64_t*>(bcast)[i] = tag(0, 0xffffffffu);
          }
        }
        s_flag = ok ? 0 : 2;
        s_r = Words<F>::load(cw);
        if (tr0) trace[j * 8 + 4] = globaltimer();
      }
    }
    __syncthreads();
    if (s_flag == 2) return;
    r = s_r;
  }
  // final fold of the size-2 tables by the last challenge (sumcheck.py:129-130)
  if (blockIdx.x == 0) publish_finals<F, MAXK>(tabs, k, r, seq0 + (uint32_t)num_vars + 1, mb);
}

// ---------------------------------------------------------------------------
// Cluster kernel (small rounds): ONE thread-block cluster of up to 16 CTAs.
// Block partials meet in CTA 0's shared memory over DSMEM after a cluster
// barrier; CTA 0 publishes, polls the challenge and writes it into every
// CTA's shared memory; a second cluster barrier releases the next round
// (its release/acquire also orders this round's in-place table writes).
// No L2 tickets, no grid barrier.  Runs rounds [j0, num_vars); for j0 > 0 it
// starts by fetching r_{j0-1} from the mailbox (handoff from the grid kernel).
constexpr int kClusterMax = 16;
constexpr int kClusterThreads = 256;


// ---------------------------------------------------------------------------
// Paired rounds (cluster kernel, PROD2 / SUM2PROD2 over Fr).  Round j+1's raw
// sums are quadratics in the challenge r_j: with T the tables folded by
// r_0 .. r_{j-1}, h = half of round j, h' = h / 2 and the round-(j+1) pair i
// built from the quadruple a = T[i], b = T[i + h'], c = T[i + h], d =
// T[i + h + h'], its lo / hi / difference entries are p + r (q - p) for
// (p, q) = (a, c), (b, d), (b - a, d - c), and each product sum is
//   sum (p_F + r dF)(p_X + r dX) = S_pp + r (S_qq - S_pp - S_dd) + r^2 S_dd
// with S_pp = sum p_F p_X, S_qq = sum q_F q_X, S_dd = sum (q - p)_F (q - p)_X.
// Round j's own raw sums are S_pp + S_qq over the lo and hi kinds (its pairs
// are (a, c) and (b, d)).  So one pass publishes the 3 sums per raw output
// (9 or 18 wide values); the host evaluates round j, draws r_j, evaluates
// round j+1 at r_j, draws r_{j+1} and answers both (ch, ch2); the next pass
// first folds the tables twice.  One PCIe round trip per two rounds.
template <class F, class EV>
struct La {
  static constexpr bool kOn = false;
  static constexpr int NR = 1, NT = 1, L = 32;
};
template <int MAXK>
struct La<Fr255, EvProd2<Fr255, MAXK>> {
  static constexpr bool kOn = true;
  static constexpr int NR = 3, NT = 2, L = 16;  // 8 fold lanes, 9 product lanes
};
template <int MAXK>
struct La<Fr255, EvSum2Prod2<Fr255, MAXK>> {
  static constexpr bool kOn = true;
  static constexpr int NR = 6, NT = 3, L = 32;  // 12 fold lanes, 18 product lanes
};

// a wide sum of storage-form values -> its residue (storage form)
ZKL_D fr_t wide_to_field(const Red<Fr255>::W& w) {
  fr_t lo;
#pragma unroll
  for (int i = 0; i < 8; i++) lo.v[i] = w.w[i];
  lo = Fr255::reduce_once(Fr255::reduce_once(lo));  // lo < 2^256 < 3p
  if (w.w[8]) {
    fr_t h = Fr255::zero();
    h.v[0] = w.w[8];
    lo = Fr255::add(lo, Fr255::mul(h, Fr255::r2()));  // w8 2^256 mod p
  }
  return lo;
}

template <class F, int MAXK, class EV>
__global__ void __launch_bounds__(kClusterThreads)
    k_sumcheck_cluster(TablePtrs<F, MAXK> tabs, int k, int num_vars, int j0, int j_end,
                       Terms<F> tm, Mailbox* mb, unsigned* fail, uint32_t seq0, uint64_t* trace,
                       int L) {
  using T = typename F::T;
  using R = Red<F>;
  using W = typename R::W;
  constexpr int NC = Words<F>::N;
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank(), C = cluster.num_blocks();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  __shared__ W wsum[kClusterThreads / 32][EV::NOUT];
  __shared__ W s_part[EV::NOUT];           // this CTA's partial (read by CTA 0)
  __shared__ T s_r;                        // challenge (written by CTA 0)
  __shared__ int s_flag;
  __shared__ uint64_t s_words[kMbEvalWords];
  const uint64_t nthreads = (uint64_t)C * blockDim.x;
  const uint64_t gtid = rank * (uint64_t)blockDim.x + threadIdx.x;
  T r = F::zero();
  // CTA 0 thread 0: poll r_{seq-1} and hand it to every CTA (then barrier)
  __shared__ uint32_t s_cw[NC];
  auto fetch_challenge = [&](uint32_t seq) {
    if (rank == 0 && warp == 0) {
      const bool ok = warp_poll<NC>(mb->ch, seq, s_cw, &mb->abort);
      if (lane == 0) {
        if (!ok) {
          *fail = 1;
          mb->status = 1;
        }
        s_r = Words<F>::load(s_cw);
        s_flag = ok ? 0 : 2;
      }
      __syncwarp();
      if (lane < (int)C) {  // lane b copies into CTA b
        *cluster.map_shared_rank(&s_r, lane) = s_r;
        *cluster.map_shared_rank(&s_flag, lane) = s_flag;
      }
    }
    cluster.sync();
  };
  if (j0 > 0) {
    fetch_challenge(seq0 + (uint32_t)j0);
    if (s_flag == 2) return;
    r = s_r;
  }
  // one round evaluated directly: fold by r, evaluate, reduce, publish
  auto direct_round = [&](int j) {
    const uint32_t seq = seq0 + (uint32_t)j + 1;
    const bool fold = j > 0;
    const bool tr0 = trace && rank == 0 && threadIdx.x == 0;
    if (tr0) trace[j * 8 + 0] = globaltimer();
    const uint64_t tb0 = trace ? globaltimer() : 0;
    const uint64_t half = 1ull << (num_vars - 1 - j);
    // lane mode while a round needs at most (L >> 8) & 255 passes of the cluster
    const int Ll = L & 255;
    const int Lr =
        (Ll > 0 && half * (uint64_t)Ll <= nthreads * (uint64_t)((L >> 8) & 255)) ? Ll : 0;
    accumulate_round<F, MAXK, EV>(tabs, k, tm, half, fold, r, Lr, gtid, nthreads, wsum);
    if (tr0) trace[j * 8 + 1] = globaltimer();
    __syncthreads();
    if (trace && threadIdx.x == 0) {  // per-block accumulate time and SM (ZKL_TRACE)
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trace[(size_t)num_vars * 8 + ((size_t)j * gridDim.x + blockIdx.x) * 2] = globaltimer() - tb0;
      trace[(size_t)num_vars * 8 + ((size_t)j * gridDim.x + blockIdx.x) * 2 + 1] = smid;
    }
    if (warp == 0) {
      W v[EV::NOUT];
      block_total<F, EV::NOUT>(wsum, nwarps, v);
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < EV::NOUT; q++) s_part[q] = v[q];
      }
    }
    cluster.sync();  // every CTA's partial is in its shared memory
    if (tr0) trace[j * 8 + 2] = globaltimer();
    if (rank == 0 && warp == 0) {
      W tot[EV::NOUT];
#pragma unroll
      for (int q = 0; q < EV::NOUT; q++) {
        W pv = lane < (int)C ? *cluster.map_shared_rank(&s_part[q], lane) : R::zero();
#pragma unroll
        for (int off = 16; off; off >>= 1) pv = R::add(pv, R::shfl_down(pv, off));
        tot[q] = pv;
      }
      publish_sums<F, EV::NOUT>(tot, seq, mb, s_words);
      if (trace && lane == 0) trace[j * 8 + 3] = globaltimer();
    }
  };
  int jl = j0;  // first round of the direct loop
  if constexpr (La<F, EV>::kOn) {
    // paired rounds (host flag; j_end < num_vars: a host tail follows)
    if (((L >> 16) & 1) && j0 == 0 && j_end >= 2 && j_end < num_vars) {
      using LA = La<F, EV>;
      constexpr int NP = 3 * LA::NR;  // product sums per pass
      constexpr int Lq = LA::L;
      __shared__ W la_wsum[kClusterThreads / 32][NP];
      __shared__ W la_gather[kClusterMax][NP];
      __shared__ T s_r2;  // r_{j+1} of a pair (written by CTA 0)
      __shared__ uint32_t s_cw2[NC];
      const int tF = tm.fi[0][0], tG = tm.fi[0][1], tH = LA::NT == 3 ? tm.fi[1][1] : 0;
      auto tab_of = [&](int t) -> T* { return tabs.t[t == 0 ? tF : t == 1 ? tG : tH]; };
      // one pass over round j's quadruples (round j+1's pairs): the tables are
      // first brought from round j-2 to round j by folding with (ra, rb) when
      // `fold`; then the 3 NR product sums, reduced over the cluster and
      // published under round j's tag
      auto la_pass = [&](int j, int nfold, const T& ra, const T& rb) {
        const uint64_t h1 = 1ull << (num_vars - 2 - j);  // pairs of round j+1
        const uint64_t hj = 2 * h1;                      // round j's half
        const uint64_t hm1 = 2 * hj, hm2 = 4 * hj;       // rounds j-1, j-2 halves
        const uint64_t ngroups = nthreads / Lq;
        const int q = lane & (Lq - 1), gb = lane & ~(Lq - 1);
        // fold lane q < 4 NT: table q / 4, entry q % 4 of the quadruple (a, b, c, d)
        const bool fl = q < 4 * LA::NT;
        T* tq = tab_of(fl ? q >> 2 : 0);
        const uint64_t moff = (uint64_t)(q & 1) * h1 + (uint64_t)((q >> 1) & 1) * hj;
        // product lane q < 3 NR: raw output o = q / 3 (F x G for o < 3, F x H
        // above), kind 0 lo (a, c), 1 hi (b, d), 2 difference (b - a, d - c);
        // term sk: 0 p p, 1 q q, 2 (q - p)(q - p)
        const bool pl = q < NP;
        const int o = pl ? q / 3 : 0, sk = q % 3, kind = o % 3;
        const int xl = o < 3 ? 4 : 8;
        T acc = F::zero();
        const uint64_t passes = (h1 + ngroups - 1) / ngroups;
        uint64_t i = gtid / Lq;
        for (uint64_t ps = 0; ps < passes; ps++, i += ngroups) {
          const bool active = i < h1;
          T v = F::zero();
          if (active && fl) {
            const uint64_t m = i + moff;
            if (nfold == 2) {  // T_j[m] from T_{j-2}: two folds by ra, then one by rb
              const T x0 = ld_cg(tq + m), x1 = ld_cg(tq + m + hm2);
              const T y0 = ld_cg(tq + m + hm1), y1 = ld_cg(tq + m + hm1 + hm2);
              const T u0 = F::add(x0, F::mul(ra, F::sub(x1, x0)));
              const T u1 = F::add(y0, F::mul(ra, F::sub(y1, y0)));
              v = F::add(u0, F::mul(rb, F::sub(u1, u0)));
              tq[m] = v;
            } else if (nfold == 1) {  // T_j[m] from T_{j-1} by ra
              const T x0 = ld_cg(tq + m), x1 = ld_cg(tq + m + hm1);
              v = F::add(x0, F::mul(ra, F::sub(x1, x0)));
              tq[m] = v;
            } else {
              v = ld_cg(tq + m);
            }
          }
          const T fa = shfl_elem<F>(v, gb), fb = shfl_elem<F>(v, gb + 1);
          const T fc = shfl_elem<F>(v, gb + 2), fd = shfl_elem<F>(v, gb + 3);
          const T xa = shfl_elem<F>(v, gb + xl), xb = shfl_elem<F>(v, gb + xl + 1);
          const T xc = shfl_elem<F>(v, gb + xl + 2), xd = shfl_elem<F>(v, gb + xl + 3);
          T pF, qF, pX, qX;
          if (kind == 0) {
            pF = fa; qF = fc; pX = xa; qX = xc;
          } else if (kind == 1) {
            pF = fb; qF = fd; pX = xb; qX = xd;
          } else {
            pF = F::sub(fb, fa); qF = F::sub(fd, fc); pX = F::sub(xb, xa); qX = F::sub(xd, xc);
          }
          const T u = sk == 0 ? pF : sk == 1 ? qF : F::sub(qF, pF);
          const T w = sk == 0 ? pX : sk == 1 ? qX : F::sub(qX, pX);
          const T prod = F::mul(u, w);
          if (active && pl) acc = F::add(acc, prod);
        }
        W wv = R::from(acc);
#pragma unroll
        for (int off = 16; off >= Lq; off >>= 1) wv = R::add(wv, R::shfl_down(wv, off));
        if (lane < NP) la_wsum[warp][lane] = wv;
        __syncthreads();
        if (warp == 0 && lane < NP) {
          W t = la_wsum[0][lane];
          for (int w2 = 1; w2 < nwarps; w2++) t = R::add(t, la_wsum[w2][lane]);
          *cluster.map_shared_rank(&la_gather[rank][lane], 0) = t;
        }
        cluster.sync();
        if (rank == 0 && warp == 0) {  // lane p: product p over the cluster, tagged words
          const uint32_t seq = seq0 + (uint32_t)j + 1;
          if (lane < NP) {
            W t = la_gather[0][lane];
            for (unsigned c2 = 1; c2 < C; c2++) t = R::add(t, la_gather[c2][lane]);
#pragma unroll
            for (int w = 0; w < R::NW; w++) s_words[lane * R::NW + w] = tag(R::word(t, w), seq);
          }
          __syncwarp();
          constexpr int NWORDS = NP * R::NW;
          for (int idx = 2 * lane; idx < NWORDS; idx += 64) {
            if (idx + 1 < NWORDS)
              st_tagged2(mb->ev + idx, s_words[idx], s_words[idx + 1]);
            else
              mb->ev[idx] = s_words[idx];
          }
        }
      };
      // the second challenge of a pair (ch2), read by CTA 0 and broadcast
      // a pair's two challenges (ch: r_j under tag seq, ch2: r_{j+1} under
      // seq + 1) in one poll, broadcast to every CTA
      auto fetch_pair = [&](uint32_t seq) {
        if (rank == 0 && warp == 0) {
          const bool ok = warp_poll2<NC>(mb->ch, mb->ch2, seq, s_cw, s_cw2, &mb->abort);
          if (lane == 0) {
            if (!ok) {
              *fail = 1;
              mb->status = 1;
            }
            s_r = Words<F>::load(s_cw);
            s_r2 = Words<F>::load(s_cw2);
            s_flag = ok ? 0 : 2;
          }
          __syncwarp();
          if (lane < (int)C) {
            *cluster.map_shared_rank(&s_r, lane) = s_r;
            *cluster.map_shared_rank(&s_r2, lane) = s_r2;
            *cluster.map_shared_rank(&s_flag, lane) = s_flag;
          }
        }
        cluster.sync();
      };
      // rounds before jp (more quadruples than (L >> 17) cluster passes) run
      // directly; the host derives the same jp
      const uint64_t pp = (uint64_t)((L >> 17) & 127);
      int j = 0;
      while (j < j_end && (1ull << (num_vars - 2 - j)) * (uint64_t)Lq > nthreads * pp) j++;
      if ((j_end - j) & 1) j++;  // whole pairs only: an odd one out runs directly
      for (int jd = 0; jd < j; jd++) {
        direct_round(jd);
        fetch_challenge(seq0 + (uint32_t)jd + 1);
        if (s_flag == 2) return;
        r = s_r;
      }
      T ra = r, rb = F::zero();
      int nfold = j > 0 ? 1 : 0;  // folds the tables lag behind (by ra, rb)
      bool pending = false;       // after the loop: the last pair's folds
      while (j < j_end) {
        const bool tr0 = trace && rank == 0 && threadIdx.x == 0;
        if (tr0) trace[j * 8 + 0] = globaltimer();
        const bool paired = j + 1 < j_end;
        la_pass(j, nfold, ra, rb);
        if (tr0) trace[j * 8 + 3] = globaltimer();
        if (paired)
          fetch_pair(seq0 + (uint32_t)j + 1);
        else
          fetch_challenge(seq0 + (uint32_t)j + 1);
        if (s_flag == 2) return;
        if (paired) {
          ra = s_r;
          rb = s_r2;
          nfold = 2;
          pending = true;
          j += 2;
        } else {
          r = s_r;
          pending = false;
          j += 1;
        }
        if (tr0) trace[(j - 1) * 8 + 4] = globaltimer();
      }
      if (pending) {
        // the last pair's two folds fused into the host tail's mail: survivor
        // i of table q from the four entries i, i + hb, i + ha, i + ha + hb of
        // the round-(j_end - 2) table (ha, hb: rounds j_end - 2, j_end - 1 halves)
        const uint64_t hb = 1ull << (num_vars - j_end), ha = 2 * hb;
        const uint32_t fseq = seq0 + (uint32_t)num_vars + 1;
        for (uint64_t idx = gtid; idx < (uint64_t)k * hb; idx += nthreads) {
          const int q = (int)(idx / hb);
          const uint64_t i = idx - (uint64_t)q * hb;
          const T* t = tabs.t[q];
          const T x0 = ld_cg(t + i), x1 = ld_cg(t + i + ha);
          const T y0 = ld_cg(t + i + hb), y1 = ld_cg(t + i + hb + ha);
          const T u0 = F::add(x0, F::mul(ra, F::sub(x1, x0)));
          const T u1 = F::add(y0, F::mul(ra, F::sub(y1, y0)));
          const T f = F::add(u0, F::mul(rb, F::sub(u1, u0)));
#pragma unroll
          for (int w = 0; w < NC; w++) mb->tail[idx * NC + w] = tag(Words<F>::word(f, w), fseq);
        }
        return;
      }
      jl = j_end;
    }
  }
  for (int j = jl; j < j_end; j++) {
    direct_round(j);
    const uint32_t seq = seq0 + (uint32_t)j + 1;
    const bool tr0 = trace && rank == 0 && threadIdx.x == 0;
    fetch_challenge(seq);
    if (tr0) trace[j * 8 + 4] = globaltimer();
    if (s_flag == 2) return;
    r = s_r;
  }
  if (j_end == num_vars) {
    if (rank == 0) publish_finals<F, MAXK>(tabs, k, r, seq0 + (uint32_t)num_vars + 1, mb);
    return;
  }
  // host tail: fold by the last challenge and send the k x 2^(n - j_end)
  // survivors to the host as tagged words (it runs the remaining rounds)
  const uint64_t th = 1ull << (num_vars - j_end);
  const uint32_t fseq = seq0 + (uint32_t)num_vars + 1;
  for (uint64_t idx = gtid; idx < (uint64_t)k * th; idx += nthreads) {
    const int q = (int)(idx / th);
    const uint64_t i = idx - (uint64_t)q * th;
    const T* t = tabs.t[q];
    const T a = ld_cg(t + i), b = ld_cg(t + i + th);
    const T f = F::add(a, F::mul(r, F::sub(b, a)));
#pragma unroll
    for (int w = 0; w < NC; w++) mb->tail[idx * NC + w] = tag(Words<F>::word(f, w), fseq);
  }
}

// ---------------------------------------------------------------------------
// Launch planning.  A Montgomery product is ~500 SASS instructions, so a
// round whose pairs all fit in one wave is issue-bound per SM sub-partition,
// not memory-bound: spread large rounds over many SMs with few warps each
// (block size = ceil(threads / SMs) rounded to a warp, 32..256), and run the
// small rounds (threads <= one cluster) in the cluster kernel.
inline int block_for(uint64_t threads, int sms) {
  uint64_t per_sm = (threads + sms - 1) / sms;
  uint64_t bs = (per_sm + 31) / 32 * 32;
  if (bs < 32) bs = 32;
  if (bs > (uint64_t)kThreads) bs = kThreads;
  return (int)bs;
}

struct Plan {
  int j_switch;      // rounds [0, j_switch) grid kernel, [j_switch, n) cluster kernel
  int grid, block;   // grid kernel shape
  int cgrid, cblock; // cluster kernel shape (one cluster)
  int lanes;
  int j_end;         // cluster kernel stops after round j_end - 1 (host tail below n)
  int la_np;         // paired rounds: product sums per pass (0 = one round per trip)
};

template <class F, int MAXK, class EV>
struct Persistent {
  static int launch_grid(const Plan& pl, void* const* tables, int k, int num_vars,
                         const Terms<F>& tm, Mailbox* mb, typename Red<F>::W* partials,
                         unsigned* ticket, uint64_t* bcast, unsigned* fail, uint32_t seq0,
                         uint64_t* trace, cudaStream_t s) {
    TablePtrs<F, MAXK> tp;
    for (int j = 0; j < MAXK; j++) tp.t[j] = j < k ? (typename F::T*)tables[j] : nullptr;
    Terms<F> tmc = tm;
    static const unsigned direct_max = [] {
      const char* e = getenv("ZKL_DIRECT_POLL_MAX");
      return e ? (unsigned)atoi(e) : (unsigned)kDirectPollMaxGrid;
    }();
    int direct = (unsigned)pl.grid <= direct_max ? 1 : 0;
    int L = pl.lanes, j0 = 0, j1 = pl.j_switch;
    void* args[] = {&tp, &k, &num_vars, &j0, &j1, &tmc, &mb, &partials, &ticket, &bcast,
                    &fail, &seq0, &direct, &trace, &L};
    ZKL_CUDA(cudaLaunchCooperativeKernel((const void*)k_sumcheck_persistent<F, MAXK, EV>,
                                         pl.grid, pl.block, args, 0, s));
    ZKL_LAUNCH_CHECK();
    return kOk;
  }
  static int launch_cluster(const Plan& pl, void* const* tables, int k, int num_vars,
                            const Terms<F>& tm, Mailbox* mb, unsigned* fail, uint32_t seq0,
                            uint64_t* trace, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
      ZKL_CUDA(cudaFuncSetAttribute((const void*)k_sumcheck_cluster<F, MAXK, EV>,
                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      attr = true;
    }
    TablePtrs<F, MAXK> tp;
    for (int j = 0; j < MAXK; j++) tp.t[j] = j < k ? (typename F::T*)tables[j] : nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.cgrid);
    cfg.blockDim = dim3(pl.cblock);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pl.cgrid;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static const int passes = [] {  // ZKL_CLUSTER_LANE_PASSES (default 4)
      const char* e = getenv("ZKL_CLUSTER_LANE_PASSES");
      const int v = e ? atoi(e) : 4;
      return v < 1 ? 1 : v > 64 ? 64 : v;
    }();
    static const int pair_passes = [] {  // ZKL_PAIR_PASSES (run_phase reads the same)
      const char* e = getenv("ZKL_PAIR_PASSES");
      const int v = e ? atoi(e) : 1;
      return v < 1 ? 1 : v > 127 ? 127 : v;
    }();
    const int lp = pl.lanes | (passes << 8) |
                   (La<F, EV>::kOn && pl.la_np ? (1 << 16) | (pair_passes << 17) : 0);
    ZKL_CUDA(cudaLaunchKernelEx(&cfg, k_sumcheck_cluster<F, MAXK, EV>, tp, k, num_vars,
                                pl.j_switch, pl.j_end, tm, mb, fail, seq0, trace, lp));
    ZKL_LAUNCH_CHECK();
    return kOk;
  }
  static Plan plan(int num_vars, int lanes) {
    static int per_sm = -1, sms = kSMs;
    if (per_sm < 0) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
              &per_sm, k_sumcheck_persistent<F, MAXK, EV>, kThreads, 0) != cudaSuccess ||
          per_sm < 1)
        per_sm = 1;
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    Plan pl;
    pl.lanes = lanes;
    pl.j_end = num_vars;
    pl.la_np = 0;
    const uint64_t per_pair = lanes > 0 ? (uint64_t)lanes : 1;
    // cluster: up to 16 CTAs x 256 threads; lane mode loops when a round
    // has more pairs than lane groups (at most kClusterPasses passes)
    const uint64_t cap = (uint64_t)kClusterMax * kClusterThreads;
    const uint64_t kClusterPasses = 4;
    int js = 0;
    while (js < num_vars && (1ull << (num_vars - 1 - js)) * per_pair > cap * kClusterPasses) js++;
    pl.j_switch = js;
    const uint64_t want_c = (1ull << (num_vars - 1 - js)) * per_pair;  // threads, round js
    int cb = kClusterThreads, cg_ = kClusterMax;
    if (want_c < cap) {  // shrink: fewer CTAs first, then fewer threads
      cg_ = (int)((want_c + kClusterThreads - 1) / kClusterThreads);
      if (cg_ < 1) cg_ = 1;
      if (cg_ == 1) {
        cb = (int)((want_c + 31) / 32 * 32);
        if (cb < 32) cb = 32;
      }
    }
    pl.cgrid = cg_;
    pl.cblock = cb;
    const uint64_t want = (1ull << (num_vars - 1)) * per_pair;
    const int bs = block_for(want, sms);
    pl.block = bs;
    uint64_t gcap = (uint64_t)sms * per_sm * (kThreads / bs);
    if (gcap > 65535) gcap = 65535;
    uint64_t g = (want + bs - 1) / bs;
    pl.grid = (int)(g < 1 ? 1 : (g > gcap ? gcap : g));
    return pl;
  }
};

template <class F>
int detect_shape(const Terms<F>& tm) {
  if (tm.nterms == 1 && tm.nf[0] == 2 && tm.degree >= 2) return kProd2;
  if (tm.nterms == 1 && tm.nf[0] == 3 && tm.degree == 3) return kProd3;
  if (tm.nterms == 2 && tm.nf[0] == 2 && tm.nf[1] == 2 && tm.fi[0][0] == tm.fi[1][0] &&
      tm.degree >= 2)
    return kSum2Prod2;
  if (tm.nterms == 2 && tm.nf[0] == 3 && tm.nf[1] == 2 && tm.fi[1][0] == tm.fi[0][0] &&
      tm.degree == 3)
    return kZkMat;
  if (tm.nterms == 5 && tm.degree == 3 && tm.nf[0] == 3 && tm.nf[1] == 2 && tm.nf[2] == 3 &&
      tm.nf[3] == 1 && tm.nf[4] == 2 && tm.fi[1][0] == tm.fi[0][0] &&
      tm.fi[2][0] == tm.fi[0][0] && tm.fi[3][0] == tm.fi[0][1] && tm.fi[4][1] == tm.fi[2][1])
    return kLogup;
  return kGeneric;
}

template <class F>
struct LaunchReq {
  int shape, k, num_vars;
  void* const* tables;
  const Terms<F>* tm;
  Mailbox* mb;
  typename Red<F>::W* partials;
  unsigned *ticket, *fail;
  uint64_t* bcast;
  uint32_t seq0;
  uint64_t* trace;
  cudaStream_t s;
};

// query (pl != null, launch == false): fill the plan; launch: both kernels
// launch: 0 = plan only, 1 = the grid kernel (rounds [0, j_switch)),
// 2 = the cluster kernel (rounds [j_switch, n)).  The host launches the
// cluster part only once the grid kernel no longer waits on it (at the
// handoff round): a launch that blocks -- e.g. lazy loading of the kernel
// image on first use -- must never sit between a device kernel and the host
// answer it is spinning for.
template <class F, int MAXK>
static int dispatch(const LaunchReq<F>& q, Plan* pl, int* nout, int launch) {
#define ZKL_SHAPE(EVT)                                                                      \
  {                                                                                         \
    using P = Persistent<F, MAXK, EVT<F, MAXK>>;                                            \
    *nout = EVT<F, MAXK>::NOUT;                                                             \
    if (!launch) {                                                                          \
      *pl = P::plan(q.num_vars, lanes_for(q.shape, q.k));                                  \
      return kOk;                                                                           \
    }                                                                                       \
    if (launch == 1)                                                                        \
      return P::launch_grid(*pl, q.tables, q.k, q.num_vars, *q.tm, q.mb, q.partials,        \
                            q.ticket, q.bcast, q.fail, q.seq0, q.trace, q.s);               \
    return P::launch_cluster(*pl, q.tables, q.k, q.num_vars, *q.tm, q.mb, q.fail, q.seq0,   \
                             q.trace, q.s);                                                 \
  }
  switch (q.shape) {
    case kProd2: ZKL_SHAPE(EvProd2)
    case kProd3: ZKL_SHAPE(EvProd3)
    case kSum2Prod2: ZKL_SHAPE(EvSum2Prod2)
    case kZkMat:
      if constexpr (MAXK >= 4) ZKL_SHAPE(EvZkMat)
      else ZKL_SHAPE(EvGeneric)
    case kLogup:
      if constexpr (MAXK >= 8) ZKL_SHAPE(EvLogup)
      else ZKL_SHAPE(EvGeneric)
    case kLogupTiled:
      if constexpr (MAXK >= 4) ZKL_SHAPE(EvLogupTiled)
      else ZKL_SHAPE(EvGeneric)
    default: ZKL_SHAPE(EvGeneric)
  }
#undef ZKL_SHAPE
}

template <class F>
static int run_dispatch(const LaunchReq<F>& q, Plan* pl, int* nout, int launch) {
  if (q.k <= 2) return dispatch<F, 2>(q, pl, nout, launch);
  if (q.k <= 4) return dispatch<F, 4>(q, pl, nout, launch);
  return dispatch<F, 8>(q, pl, nout, launch);
}

// ---------------------------------------------------------------------------
// host side
template <class F>
struct HostRed;
template <>
struct HostRed<Fr255> {
  // words: 9 x u32 = lo (256 bits) + w8 * 2^256 -> residue (storage form)
  static fr_t reduce(const uint32_t* w) {
    fr_t lo;
    memcpy(&lo, w, 32);
    for (int k = 0; k < 2; k++)  // lo < 2^256 < 3p
      if (Fr255::geq_p_portable(lo)) lo = Fr255::sub_p_portable(lo);
    if (w[8] == 0) return lo;
    fr_t h = Fr255::zero();
    h.v[0] = w[8];
    h = host::Fr::mul(h, Fr255::r2());  // w8 * 2^256 mod p
    return host::Fr::add(lo, h);
  }
};
template <>
struct HostRed<M61> {
  static uint64_t reduce(const uint32_t* w) {
    const unsigned __int128 v =
        ((unsigned __int128)(((uint64_t)w[3] << 32) | w[2]) << 64) | (((uint64_t)w[1] << 32) | w[0]);
    return (uint64_t)(v % M61::P);
  }
};

template <class F>
static bool mailbox_ready(const volatile uint64_t* src, int nwords, uint32_t seq, uint32_t* out) {
  for (int i = 0; i < nwords; i++) {
    const uint64_t v = src[i];
    if ((uint32_t)(v >> 32) != seq) return false;
    out[i] = (uint32_t)v;
  }
  return true;
}

template <class F>
static int wait_words(Mailbox* mb, const volatile uint64_t* src, int nwords, uint32_t seq,
                      uint32_t* out, cudaStream_t s, const char* what, int round) {
  const auto until = std::chrono::steady_clock::now() + std::chrono::seconds(30);
  uint64_t spins = 0;
  while (!mailbox_ready<F>(src, nwords, seq, out)) {
    if ((++spins & 0xffff) == 0) {
      if (mb->status) {
        set_error("persistent sumcheck: device gave up waiting (round %d)", round);
        return kErrCuda;
      }
      cudaError_t q = cudaStreamQuery(s);
      if (q != cudaErrorNotReady && !mailbox_ready<F>(src, nwords, seq, out)) {
        set_error("persistent sumcheck ended before publishing %s of round %d: %s", what, round,
                  cudaGetErrorString(q == cudaSuccess ? cudaErrorUnknown : q));
        return kErrCuda;
      }
      if (std::chrono::steady_clock::now() > until) {
        mb->abort = 1;
        cudaStreamSynchronize(s);
        set_error("persistent sumcheck: device did not publish %s of round %d", what, round);
        return kErrCuda;
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return kOk;
}

template <class F>
static void host_quad(const typename F::T& c0, const typename F::T& c1, const typename F::T& c2,
                      typename F::T* out) {
  using H = typename host::For<F>::H;
  using T = typename F::T;
  const T two_c1 = H::add(c1, c1), two_c2 = H::add(c2, c2);
  out[0] = c0;
  out[1] = c1;
  out[2] = H::sub(H::add(two_c1, two_c2), c0);
  const T six_c2 = H::add(H::add(two_c2, two_c2), two_c2);
  out[3] = H::sub(H::add(H::add(two_c1, c1), six_c2), H::add(c0, c0));
}

static bool g_phase_dirty = true;  // after a failure the ticket / flags need a reset

int host_tail_default() {
  static const int v = [] {
    const char* e = getenv("ZKL_HOST_TAIL");
    return e ? atoi(e) : 5;
  }();
  return v;
}

bool no_persistent() {
  // ncu marks its target with NV_NSIGHT_INJECTION_* / NV_TPS_LAUNCH_TOKEN;
  // compute-sanitizer and other injectors use CUDA_INJECTION64_PATH.
  // ZKL_FORCE_PERSISTENT=1 keeps the persistent engine under an injector that
  // does not replay kernels (compute-sanitizer memcheck / racecheck: the host
  // still answers every round, just slowly)
  if (getenv("ZKL_FORCE_PERSISTENT") != nullptr) return false;
  static const bool v =
      getenv("ZKL_NO_PERSISTENT") != nullptr || getenv("CUDA_INJECTION64_PATH") != nullptr ||
      getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr ||
      getenv("NV_TPS_LAUNCH_TOKEN") != nullptr ||
      (getenv("CUDA_LAUNCH_BLOCKING") && getenv("CUDA_LAUNCH_BLOCKING")[0] == '1');
  return v;
}

// the same phase, one kernel launch per round (k_round) with the host
// transcript in between; identical outputs
template <class F>
static int run_phase_stepwise(PhaseArgs<F>& a, HostTranscript& tr, uint8_t* rounds_out,
                              uint8_t* point_out, typename F::T* finals_out, cudaStream_t s) {
  using T = typename F::T;
  constexpr int nb = F::kBytes;
  a.stepwise = true;
  std::vector<T> lazy;
  if (a.prepare) {
    int rc = a.prepare(lazy);
    if (rc) return rc;
    if (!lazy.empty()) a.post_add = lazy.data();
  }
  uint64_t size = 1ull << a.num_vars;
  T r_prev = F::zero();
  for (int j = 0; j < a.num_vars; j++) {
    Post<F> post;
    post.add = a.post_add ? a.post_add[j] : F::zero();
    post.mul = a.post_mul;
    uint8_t* rj = rounds_out + (size_t)j * (a.tm.degree + 1) * nb;
    int rc = op_sumcheck_round<F>(a.tables, a.k, size, j > 0, r_prev, a.tm, post, rj, s);
    if (rc) return rc;
    if (j > 0) size >>= 1;
    for (int x = 0; x <= a.tm.degree; x++) tr.append_elem("sumcheck/eval", rj + x * nb, nb);
    challenge_canon<F>(tr, "sumcheck/round", point_out + (size_t)j * nb);
    r_prev = host::from_canon<F>(point_out + (size_t)j * nb);
  }
  std::vector<uint8_t> fc((size_t)a.k * nb);
  int rc = op_sumcheck_finish<F>(a.tables, a.k, r_prev, fc.data(), s);
  if (rc) return rc;
  a.fin_cache.resize(a.k);
  for (int q = 0; q < a.k; q++) a.fin_cache[q] = host::from_canon<F>(fc.data() + (size_t)q * nb);
  if (finals_out)
    for (int q = 0; q < a.k; q++) finals_out[q] = a.fin_cache[q];
  return kOk;
}

template <class F>
int wait_phase_finals(const PhaseArgs<F>& a, typename F::T* finals_out, cudaStream_t s) {
  constexpr int NC = Words<F>::N;
  if (a.stepwise || a.host_done) {
    for (int q = 0; q < a.k; q++) finals_out[q] = a.fin_cache[q];
    return kOk;
  }
  Mailbox* mb_host;
  Mailbox* mb_dev;
  int rc = mailbox_for_current_device(&mb_host, &mb_dev);
  if (rc) return rc;
  uint32_t fw[kMbFinalWords];
  rc = wait_words<F>(mb_host, mb_host->fin, a.k * NC, a.seq0 + a.num_vars + 1, fw, s, "finals",
                     a.num_vars);
  if (rc) {
    g_phase_dirty = true;
    return rc;
  }
  for (int q = 0; q < a.k; q++) memcpy(&finals_out[q], fw + q * NC, F::kBytes);
  return kOk;
}

template <class F>
static int run_phase_replay(PhaseArgs<F>& a, HostTranscript& tr, uint8_t* rounds_out,
                            uint8_t* point_out, typename F::T* finals_out, cudaStream_t s);

// The last n - ndev rounds of a phase on the host (PhaseArgs::host_tail):
// the cluster kernel has folded by r_{ndev-1} and sent the k x 2^(n-ndev)
// survivors; each round evaluates
//   evals[x] = post_mul (post_add[j] + sum_i sum_t coef_t prod_f T_f(x, i)),
// T(x, i) = T[i] + x (T[i + half] - T[i]), exactly the device identities,
// then appends / draws as the device loop does and folds by the challenge.
template <class F>
static int host_tail_rounds(PhaseArgs<F>& a, Mailbox* mb_host, uint32_t seq0, int ndev,
                            const typename F::T* post_add, const typename F::T& pm,
                            HostTranscript& tr, uint8_t* rounds_out, uint8_t* point_out,
                            cudaStream_t s) {
  using T = typename F::T;
  using H = typename host::For<F>::H;
  constexpr int NC = Words<F>::N, nb = F::kBytes;
  const Terms<F>& tm = a.tm;
  const int n = a.num_vars, k = a.k, deg = tm.degree;
  static const bool tracing = getenv("ZKL_TRACE") != nullptr;
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
  };
  const double t0 = tracing ? now_us() : 0;
  uint64_t cur = 1ull << (n - ndev);
  std::vector<uint32_t> words((size_t)k * cur * NC);
  int rc = wait_words<F>(mb_host, mb_host->tail, (int)words.size(), seq0 + (uint32_t)n + 1,
                         words.data(), s, "tail tables", ndev);
  if (rc) return rc;
  const double t1 = tracing ? now_us() : 0;
  std::vector<T> tab((size_t)k * cur);
  for (size_t i = 0; i < tab.size(); i++) memcpy(&tab[i], words.data() + i * NC, nb);
  const uint64_t stride = cur;  // table q at tab[q * stride ..]
  // per term: a 2-factor product needs 3 sums (f0 g0, f1 g1, fd gd; x = 2, 3
  // follow from the quadratic), a linear term 2, a 3-factor product 4
  std::vector<T> lo((size_t)k), hi((size_t)k), df((size_t)k);
  for (int j = ndev; j < n; j++) {
    const uint64_t half = cur >> 1;
    T acc[kMaxTerms][4];
    for (int t = 0; t < tm.nterms; t++)
      for (int x = 0; x < 4; x++) acc[t][x] = H::zero();
    for (uint64_t i = 0; i < half; i++) {
      for (int q = 0; q < k; q++) {
        lo[q] = tab[q * stride + i];
        hi[q] = tab[q * stride + i + half];
        df[q] = H::sub(hi[q], lo[q]);
      }
      for (int t = 0; t < tm.nterms; t++) {
        const int* fi = tm.fi[t];
        switch (tm.nf[t]) {
          case 0:
            acc[t][0] = H::add(acc[t][0], H::one());
            break;
          case 1:
            acc[t][0] = H::add(acc[t][0], lo[fi[0]]);
            acc[t][1] = H::add(acc[t][1], hi[fi[0]]);
            break;
          case 2:
            acc[t][0] = H::add(acc[t][0], H::mul(lo[fi[0]], lo[fi[1]]));
            acc[t][1] = H::add(acc[t][1], H::mul(hi[fi[0]], hi[fi[1]]));
            acc[t][2] = H::add(acc[t][2], H::mul(df[fi[0]], df[fi[1]]));
            break;
          default: {
            T v0 = lo[fi[0]], v1 = lo[fi[1]], v2 = lo[fi[2]];
            for (int x = 0; x <= deg; x++) {
              if (x) {
                v0 = H::add(v0, df[fi[0]]);
                v1 = H::add(v1, df[fi[1]]);
                v2 = H::add(v2, df[fi[2]]);
              }
              acc[t][x] = H::add(acc[t][x], H::mul(H::mul(v0, v1), v2));
            }
          }
        }
      }
    }
    for (int t = 0; t < tm.nterms; t++) {
      T e[4];
      if (tm.nf[t] == 0) {  // half copies of 1 at every x
        e[0] = e[1] = e[2] = e[3] = acc[t][0];
      } else if (tm.nf[t] == 1) {
        const T d = H::sub(acc[t][1], acc[t][0]);
        e[0] = acc[t][0];
        e[1] = acc[t][1];
        e[2] = H::add(e[1], d);
        e[3] = H::add(e[2], d);
      } else if (tm.nf[t] == 2) {
        host_quad<F>(acc[t][0], acc[t][1], acc[t][2], e);
      } else {
        continue;
      }
      for (int x = 0; x < 4; x++) acc[t][x] = e[x];
    }
    uint8_t* rj = rounds_out + (size_t)j * (deg + 1) * nb;
    for (int x = 0; x <= deg; x++) {
      T v = post_add ? post_add[j] : H::zero();
      for (int t = 0; t < tm.nterms; t++) v = H::add(v, H::mul(tm.coef[t], acc[t][x]));
      host::to_canon<F>(rj + x * nb, H::mul(pm, v));
      tr.append_elem("sumcheck/eval", rj + x * nb, nb);
    }
    uint8_t rawc[64];
    tr.challenge_squeeze("sumcheck/round", 14, rawc);
    uint8_t* rcan = point_out + (size_t)j * nb;
    reduce512<F>(rawc, rcan);
    tr.challenge_absorb(rawc);
    const T r = host::from_canon<F>(rcan);
    for (int q = 0; q < k; q++)
      for (uint64_t i = 0; i < half; i++) {
        const T a0 = tab[q * stride + i];
        tab[q * stride + i] = H::add(a0, H::mul(r, H::sub(tab[q * stride + i + half], a0)));
      }
    cur = half;
  }
  a.fin_cache.resize(k);
  for (int q = 0; q < k; q++) a.fin_cache[q] = tab[q * stride];
  a.host_done = true;
  if (tracing)
    fprintf(stderr, "[zkl trace] host tail n=%d k=%d rounds %d: wait tables %.2f us, rounds %.2f us\n",
            n, k, n - ndev, t1 - t0, now_us() - t1);
  return kOk;
}

static bool profile_replay() {
  static const bool v = getenv("ZKL_PROFILE_REPLAY") != nullptr;
  return v;
}

template <class F>
int run_phase(PhaseArgs<F>& a, HostTranscript& tr, uint8_t* rounds_out, uint8_t* point_out,
              typename F::T* finals_out, cudaStream_t s) {
  if (profile_replay() && !a.replaying && !a.sharded && a.rounds_limit <= 0)
    return run_phase_replay<F>(a, tr, rounds_out, point_out, finals_out, s);
  using T = typename F::T;
  using H = typename host::For<F>::H;
  using W = typename Red<F>::W;
  constexpr int NW = Red<F>::NW, NC = Words<F>::N, nb = F::kBytes;
  const Terms<F>& tm = a.tm;
  const int n = a.num_vars, k = a.k, deg = tm.degree;
  if (k < 1 || k > kMaxTables || tm.nterms < 0 || tm.nterms > kMaxTerms || deg < 0 || deg > 3 ||
      n < 1 || n > 63) {
    set_error("sumcheck_prove: bad arguments");
    return kErrArg;
  }
  if (no_persistent() && !a.replaying)
    return run_phase_stepwise<F>(a, tr, rounds_out, point_out, finals_out, s);
  Mailbox* mb_host;
  Mailbox* mb_dev;
  int rc = mailbox_for_current_device(&mb_host, &mb_dev);
  if (rc) return rc;
  int shape = a.forced_shape >= 0 ? a.forced_shape : detect_shape<F>(tm);
  if (shape == kLogup && k <= 4) shape = kGeneric;  // built for MAXK 8
  const int nrun = a.rounds_limit > 0 ? a.rounds_limit : n;
  if (nrun < n && finals_out) {
    set_error("sumcheck phase: a partial phase has no finals");
    return kErrArg;
  }
  LaunchReq<F> rq;
  rq.shape = shape;
  rq.k = k;
  rq.num_vars = n;
  rq.tables = a.tables;
  rq.tm = &a.tm;
  rq.s = s;
  Plan pl;
  int nout = 4;
  run_dispatch<F>(rq, &pl, &nout, 0);
  if (nrun < n) pl.j_switch = nrun;  // grid kernel only, stops after round nrun-1
  // host tail: the cluster kernel runs rounds [j_switch, n - h)
  int h = a.host_tail;
  if (h > n - 1) h = n - 1;
  while (h > 0 && (size_t)k * ((size_t)1 << h) * NC > (size_t)kMbTailWords) h--;
  if (h <= 0 || nrun < n || shape == kLogupTiled || a.sharded || a.replaying ||
      n - h <= pl.j_switch)
    h = 0;
  a.host_done = false;
  if (h) pl.j_end = n - h;
  const int ndev = n - h;  // rounds the device runs (nrun when no tail)
  // paired rounds (cluster kernel, PROD2 / SUM2PROD2 over Fr, every table in
  // one term factor, a host tail after them; ZKL_PAIRED=0 turns them off):
  // one pass publishes round j's and round j+1's sums (the latter as
  // quadratics in r_j), and one round trip carries both challenges
  static const bool paired_env = [] {
    const char* e = getenv("ZKL_PAIRED");
    return !(e && atoi(e) == 0);
  }();
  if (F::kId == Fr255::kId && paired_env && h > 0 && ndev >= 2 && pl.j_switch == 0 &&
      !a.sharded && !a.replaying && (size_t)pl.cgrid * pl.cblock >= 64) {
    const int f0 = tm.fi[0][0], f1 = tm.fi[0][1];
    if (shape == kProd2 && k == 2 && f0 != f1) pl.la_np = 9;
    if (shape == kSum2Prod2 && k == 3) {
      const int f2 = tm.fi[1][1];
      if (f0 != f1 && f0 != f2 && f1 != f2) pl.la_np = 18;
    }
  }
  // the first paired round: the one whose pass fits ZKL_PAIR_PASSES (default
  // 1) cluster passes (the kernel derives the same); earlier rounds direct
  static const int pair_passes = [] {
    const char* e = getenv("ZKL_PAIR_PASSES");
    const int v = e ? atoi(e) : 1;
    return v < 1 ? 1 : v > 127 ? 127 : v;
  }();
  int jp = 0;
  if (pl.la_np) {
    const uint64_t lq = pl.la_np == 9 ? 16 : 32;
    const uint64_t nth = (uint64_t)pl.cgrid * pl.cblock;
    while (jp < ndev && (1ull << (n - 2 - jp)) * lq > nth * (uint64_t)pair_passes) jp++;
    if ((ndev - jp) & 1) jp++;  // whole pairs only (the kernel derives the same)
    if (jp >= ndev - 1) pl.la_np = 0;  // nothing to pair
  }
  const int la_np = pl.la_np;
  T la_sum[kMbMaxOut];  // a pair's product sums (storage form)
  uint32_t la_cw[NC] = {};  // a pair's first challenge, held until the second is drawn
  void* ws;
  rc = scratch_reserve((size_t)pl.grid * kMbMaxOut * sizeof(W), &ws, s);
  if (rc) return rc;
  void* fx;
  rc = fixed_words(&fx);
  if (rc) return rc;
  unsigned* fail = (unsigned*)((char*)fx + kFixedFail);
  unsigned* ticket = (unsigned*)((char*)fx + kFixedPhaseTicket);
  uint64_t* bcast = (uint64_t*)((char*)fx + kFixedBcast);
  if (g_phase_dirty) {
    ZKL_CUDA(cudaMemsetAsync((char*)fx + kFixedFail, 0, 4, s));
    ZKL_CUDA(cudaMemsetAsync((char*)fx + kFixedPhaseTicket, 0, 4, s));
    g_phase_dirty = false;
  }
  if (mb_host->seq > 0x7fff0000u) {  // tags wrap: restart (bcast tags too)
    ZKL_CUDA(cudaStreamSynchronize(s));
    memset((void*)mb_host, 0, sizeof(Mailbox));
    ZKL_CUDA(cudaMemsetAsync((char*)fx + kFixedBcast, 0, 8 * 8, s));
    mb_host->seq = 1;
  }
  if (mb_host->seq == 0) mb_host->seq = 1;
  const uint32_t seq0 = mb_host->seq;
  mb_host->seq = seq0 + (uint32_t)n + 2;
  mb_host->abort = 0;
  mb_host->status = 0;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  // ZKL_TRACE=1: per-round device timestamps + host handling times (stderr)
  static const bool tracing = getenv("ZKL_TRACE") != nullptr;
  uint64_t* trace = nullptr;
  std::vector<double> h_seen, h_sent;
  if (tracing) {
    ZKL_CUDA(cudaMalloc(&trace, (size_t)n * 8 * 8 + (size_t)n * 2 * 8 * 4096));
    ZKL_CUDA(cudaMemsetAsync(trace, 0, (size_t)n * 8 * 8, s));
    h_seen.resize(n);
    h_sent.resize(n);
  }
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
  };
  rq.mb = mb_dev;
  rq.partials = (W*)ws;
  rq.ticket = ticket;
  rq.fail = fail;
  rq.bcast = bcast;
  rq.seq0 = seq0;
  rq.trace = trace;
  // profiler: algorithmic bytes of the whole claim, sum over rounds of
  // k 2^(n-j) elements read and (from round 1) k 2^(n-j-1) written by the fold
  // (the tiled logUp phase moves only its 3 full-size tables; the 2^tile_log
  // table side stays in L2)
  const int k_full = shape == kLogupTiled ? 2 : k;
  const int ph = prof_open(kProfPhase, 3.0 * k_full * (double)(1ull << n) * F::kBytes,
                           (double)nrun, s);
  if (a.replaying) {
    // recorded challenges: point the device-side poll at them, launch the
    // grid kernel and (stream-ordered behind it) the cluster kernel, wait
    const uint32_t* rec = (const uint32_t*)a.replay_words;
    RecordedChallenges gr = {rec, mb_dev->ch, seq0};
    const unsigned zero = 0;
    ZKL_CUDA(cudaMemcpyToSymbolAsync(g_rec, &gr, sizeof gr, 0, cudaMemcpyHostToDevice, s));
    ZKL_CUDA(cudaMemcpyToSymbolAsync(g_rec_done, &zero, sizeof zero, 0, cudaMemcpyHostToDevice,
                                     s));
    rc = run_dispatch<F>(rq, &pl, &nout, pl.j_switch > 0 ? 1 : 2);
    if (!rc && pl.j_switch > 0 && pl.j_switch < n) rc = run_dispatch<F>(rq, &pl, &nout, 2);
    prof_close(ph, s);
    RecordedChallenges none = {nullptr, nullptr, 0};
    ZKL_CUDA(cudaMemcpyToSymbolAsync(g_rec, &none, sizeof none, 0, cudaMemcpyHostToDevice, s));
    ZKL_CUDA(cudaStreamSynchronize(s));
    return rc;
  }
  rc = run_dispatch<F>(rq, &pl, &nout, pl.j_switch > 0 ? 1 : 2);
  if (pl.j_switch == 0 || pl.j_switch >= n || nrun < n) prof_close(ph, s);  // else: at handoff
  if (rc) return rc;
  a.seq0 = seq0;
  // host-side finishing constants (canonical multipliers: mul(raw_storage,
  // K_canon) = value * K in canonical form), set at round 0 after prepare()
  T Kc[5];
  T pm = a.post_mul;
  T lq_c = H::one();  // LOGUP_TILED: C_j
  std::vector<T> lazy_add;
  bool prepared = !a.prepare;
  uint32_t words[kMbEvalWords];
  std::vector<double> h_first;
  if (tracing) h_first.resize(n);
  for (int j = 0; j < (h ? ndev : nrun); j++) {
    if (tracing) {  // first tagged word of this round visible
      const uint32_t tag = la_np && j > jp && (j - jp) % 2 ? seq0 + j : seq0 + j + 1;
      while ((uint32_t)(mb_host->ev[0] >> 32) != tag && !mb_host->status) {
      }
      h_first[j] = now_us();
    }
    const bool la_round = la_np && j >= jp;
    const bool la_first = la_round && (j - jp) % 2 == 0;  // first of a pair (or the last alone)
    if (!la_round || la_first) {
      rc = wait_words<F>(mb_host, mb_host->ev, (la_first ? la_np : nout) * NW, seq0 + j + 1,
                         words, s, "sums", j);
      if (rc) {
        g_phase_dirty = true;
        return rc;
      }
    }
    if (tracing) h_seen[j] = now_us();
    if (!prepared) {
      rc = a.prepare(lazy_add);
      if (rc) {
        mb_host->abort = 1;
        cudaStreamSynchronize(s);
        g_phase_dirty = true;
        return rc;
      }
      if (!lazy_add.empty()) a.post_add = lazy_add.data();
      prepared = true;
    }
    if (j == 0) {
      pm = a.post_mul;
      if (shape == kGeneric) {
        Kc[0] = host::canon_of<F>(pm);
      } else {
        const int nk = (shape == kLogup || shape == kLogupTiled) ? 5
                       : (shape == kSum2Prod2 || shape == kZkMat) ? 2 : 1;
        for (int t = 0; t < nk; t++) Kc[t] = host::canon_of<F>(H::mul(pm, a.tm.coef[t]));
      }
    }
    T raw[kMbMaxOut];
    if (la_round) {
      // product sums S[9b + 3 kind + term] (b: factor pair F.G / F.H; kind:
      // lo, hi, difference of round j+1's pairs; term: pp, qq, dd)
      if (la_first) {
        for (int q = 0; q < la_np; q++) la_sum[q] = HostRed<F>::reduce(words + q * NW);
        for (int b = 0; b < la_np / 9; b++)  // round j: (a, c) and (b, d) pairs
          for (int t = 0; t < 3; t++) raw[3 * b + t] = H::add(la_sum[9 * b + t], la_sum[9 * b + 3 + t]);
      } else {  // round j = (first) + 1 at r_{j-1}: pp + r (qq - pp - dd) + r^2 dd
        const T rp = host::from_canon<F>(point_out + (size_t)(j - 1) * nb);
        for (int b = 0; b < la_np / 9; b++)
          for (int kd = 0; kd < 3; kd++) {
            const T pp = la_sum[9 * b + 3 * kd], qq = la_sum[9 * b + 3 * kd + 1];
            const T dd = la_sum[9 * b + 3 * kd + 2];
            const T c1 = H::sub(H::sub(qq, pp), dd);
            raw[3 * b + kd] = H::add(pp, H::mul(rp, H::add(c1, H::mul(rp, dd))));
          }
      }
    } else {
      for (int q = 0; q < nout; q++) raw[q] = HostRed<F>::reduce(words + q * NW);
    }
    if (a.sharded) {
      // every rank's raw sums (storage form) through the shared-memory
      // all-gather; the host finishing below is linear in them
      const int G = shard_world();
      std::vector<uint8_t> all((size_t)G * nout * sizeof(T));
      rc = shard_exchange(raw, (size_t)nout * sizeof(T), all.data());
      if (rc) {
        mb_host->abort = 1;
        cudaStreamSynchronize(s);
        g_phase_dirty = true;
        return rc;
      }
      for (int q = 0; q < nout; q++) {
        T acc = H::zero();
        for (int g = 0; g < G; g++) {
          T v;
          memcpy(&v, all.data() + ((size_t)g * nout + q) * sizeof(T), sizeof(T));
          acc = H::add(acc, v);
        }
        raw[q] = acc;
      }
    }
    T ev[4];
    if (shape == kLogupTiled) {
      // EvLogupTiled: raw = [P0, P1, P2, sum a0, sum ad] (storage form)
      if (j == 0 && a.tm.inv_pair) raw[0] = raw[1] = H::one();
      T qx[4];
      host_quad<F>(raw[0], raw[1], raw[2], qx);
      const T& u = a.lq_u[j];
      const T l0 = H::sub(H::one(), u), ld = H::sub(H::add(u, u), H::one());
      T npairs = H::one();  // half / 2^tile_log
      for (int b = 0; b < n - 1 - j - a.tm.tile_log; b++) npairs = H::add(npairs, npairs);
      const T cst = H::add(a.tm.coef[1], H::mul(a.tm.coef[2], a.lq_k3));
      const T mbt = H::mul(a.tm.coef[4], H::mul(npairs, a.lq_smb));
      T lx = l0, ax = raw[3];
      for (int x = 0; x < 4; x++) {
        if (x) {
          lx = H::add(lx, ld);
          ax = H::add(ax, raw[4]);
        }
        T v = H::mul(H::mul(lq_c, lx), H::add(H::mul(a.tm.coef[0], qx[x]), cst));
        v = H::add(v, H::mul(a.tm.coef[3], ax));
        ev[x] = host::canon_of<F>(H::add(v, mbt));
      }
    } else if (shape == kProd2) {
      host_quad<F>(raw[0], raw[1], raw[2], ev);
      for (int x = 0; x < 4; x++) ev[x] = H::mul(ev[x], Kc[0]);
    } else if (shape == kZkMat) {
      T ec[4];
      host_quad<F>(raw[4], raw[5], raw[6], ec);
      for (int x = 0; x < 4; x++) ev[x] = H::add(H::mul(raw[x], Kc[0]), H::mul(ec[x], Kc[1]));
    } else if (shape == kSum2Prod2) {
      T e1[4], e2[4];
      host_quad<F>(raw[0], raw[1], raw[2], e1);
      host_quad<F>(raw[3], raw[4], raw[5], e2);
      for (int x = 0; x < 4; x++) ev[x] = H::add(H::mul(e1[x], Kc[0]), H::mul(e2[x], Kc[1]));
    } else if (shape == kLogup || shape == kLogupTiled) {
      T ei[4], mb[4];
      host_quad<F>(raw[4], raw[5], raw[6], ei);
      host_quad<F>(raw[13], raw[14], raw[15], mb);
      T ax = raw[11];  // A lo + x A slope
      for (int x = 0; x < 4; x++) {
        if (x) ax = H::add(ax, raw[12]);
        T v = H::add(H::mul(raw[x], Kc[0]), H::mul(ei[x], Kc[1]));
        v = H::add(v, H::mul(raw[7 + x], Kc[2]));
        v = H::add(v, H::mul(ax, Kc[3]));
        ev[x] = H::add(v, H::mul(mb[x], Kc[4]));
      }
    } else {
      for (int x = 0; x < 4; x++) ev[x] = H::mul(raw[x], Kc[0]);
    }
    if (a.post_add) {
      const T addc = host::canon_of<F>(H::mul(pm, a.post_add[j]));
      for (int x = 0; x < 4; x++) ev[x] = H::add(ev[x], addc);
    }
    uint8_t* rj = rounds_out + (size_t)j * (deg + 1) * nb;
    for (int x = 0; x <= deg; x++) {
      memcpy(rj + x * nb, &ev[x], nb);
      tr.append_elem("sumcheck/eval", rj + x * nb, nb);
    }
    uint8_t rawc[64];
    tr.challenge_squeeze("sumcheck/round", 14, rawc);
    uint8_t* rcan = point_out + (size_t)j * nb;
    reduce512<F>(rawc, rcan);
    const T rm = host::from_canon<F>(rcan);
    if (shape == kLogupTiled) {  // C_{j+1} = C_j ((1 - u_j) + r_j (2 u_j - 1))
      const T& u = a.lq_u[j];
      lq_c = H::mul(lq_c, H::add(H::sub(H::one(), u), H::mul(rm, H::sub(H::add(u, u), H::one()))));
    }
    uint32_t cw[NC];
    memcpy(cw, &rm, nb);
    const uint64_t tg = (uint64_t)(seq0 + j + 1) << 32;
    if (la_first && j + 1 < ndev) {
      memcpy(la_cw, cw, sizeof(cw));  // sent with the pair's second challenge
    } else if (la_round && !la_first) {
      // the device reads ch (r_{j-1}) first, then ch2 (r_j): write ch2 first
      for (int w = 0; w < NC; w++) mb_host->ch2[w] = tg | cw[w];
      const uint64_t tg1 = (uint64_t)(seq0 + j) << 32;
      for (int w = 0; w < NC; w++) mb_host->ch[w] = tg1 | la_cw[w];
    } else {
      for (int w = 0; w < NC; w++) mb_host->ch[w] = tg | cw[w];
    }
    std::atomic_thread_fence(std::memory_order_seq_cst);  // drain the store buffer now
    if (tracing) h_sent[j] = now_us();
    if (pl.j_switch > 0 && j == pl.j_switch - 1 && pl.j_switch < n && nrun == n) {
      // handoff: the grid kernel has published its last round and exits
      rc = run_dispatch<F>(rq, &pl, &nout, 2);
      prof_close(ph, s);
      if (rc) {
        g_phase_dirty = true;
        return rc;
      }
    }
    tr.challenge_absorb(rawc);
  }
  if (h) {
    rc = host_tail_rounds<F>(a, mb_host, seq0, ndev, lazy_add.empty() ? a.post_add : lazy_add.data(),
                             pm, tr, rounds_out, point_out, s);
    if (rc) {
      g_phase_dirty = true;
      return rc;
    }
  }
  if (finals_out) {
    rc = wait_phase_finals<F>(a, finals_out, s);
    if (rc) return rc;
  }
  if (tracing) {
    const int n = h ? ndev : nrun;  // rounds the device actually ran
    std::vector<uint64_t> tv((size_t)n * 8);
    cudaMemcpyAsync(tv.data(), trace, tv.size() * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (getenv("ZKL_TRACE")[0] == '3' && pl.j_switch > 0) {  // per-block accumulate times
      const int G = pl.grid, jn = pl.j_switch < n ? pl.j_switch : n;
      std::vector<uint64_t> bt((size_t)jn * G * 2);
      cudaMemcpy(bt.data(), trace + (size_t)a.num_vars * 8, bt.size() * 8, cudaMemcpyDeviceToHost);
      for (int j = 0; j < jn; j++) {
        fprintf(stderr, "[zkl trace] round %d block us (block:sm:us):", j);
        for (int b = 0; b < G; b++)
          fprintf(stderr, " %d:%d:%.0f", b, (int)bt[((size_t)j * G + b) * 2 + 1],
                  bt[((size_t)j * G + b) * 2] / 1e3);
        fprintf(stderr, "\n");
      }
    }
    cudaFree(trace);
    double acc[5] = {0}, hs = 0, loop = 0, hgap = 0, hfill = 0;
    for (int j = 0; j < n; j++) {
      hfill += h_seen[j] - h_first[j];
      if (j > 0) hgap += h_first[j] - h_sent[j - 1];
      const uint64_t* t = &tv[(size_t)j * 8];
      acc[0] += (t[1] - t[0]) / 1e3;                      // accumulate
      acc[1] += (t[2] - t[1]) / 1e3;                      // block reduce + ticket
      acc[2] += t[3] ? (t[3] - t[2]) / 1e3 : 0;           // last-block sum + publish
      acc[3] += t[4] ? (t[4] - (t[3] ? t[3] : t[2])) / 1e3 : 0;  // wait for challenge
      if (j + 1 < n && t[4]) loop += (tv[(size_t)(j + 1) * 8] - t[4]) / 1e3;
      hs += h_sent[j] - h_seen[j];
      if (getenv("ZKL_TRACE")[0] == '4')  // raw stamps t0..t4 relative (paired-round debugging)
        fprintf(stderr, "[zkl trace] la round %d: publish %.2f | passes %.2f | reduce %.2f | "
                "coef->r %.2f | host seen->sent %.2f\n", j, ((double)t[3] - (double)t[0]) / 1e3,
                ((double)t[1] - (double)t[0]) / 1e3, ((double)t[2] - (double)t[1]) / 1e3,
                ((double)t[4] - (double)t[2]) / 1e3, h_sent[j] - h_seen[j]);
      if (getenv("ZKL_TRACE")[0] == '2')
        fprintf(stderr, "[zkl trace] round %d: accum %.2f reduce %.2f publish %.2f wait %.2f\n", j,
                (t[1] - t[0]) / 1e3, (t[2] - t[1]) / 1e3, t[3] ? (t[3] - t[2]) / 1e3 : 0.0,
                t[4] ? (t[4] - (t[3] ? t[3] : t[2])) / 1e3 : 0.0);
    }
    fprintf(stderr,
            "[zkl trace] n=%d k=%d shape=%d grid=%dx%d->%d cluster=%dx%d per-round us: accum "
            "%.2f | reduce %.2f | publish %.2f | wait-challenge %.2f | to-next %.2f | host %.2f "
            "| host: sent->next-first %.2f, first->all %.2f\n",
            n, k, shape, pl.grid, pl.block, pl.j_switch, pl.cgrid, pl.cblock, acc[0] / n, acc[1] / n, acc[2] / n, acc[3] / n,
            n > 1 ? loop / (n - 1) : 0.0, hs / n, n > 1 ? hgap / (n - 1) : 0.0, hfill / n);
  }
  return kOk;
}

// ZKL_PROFILE_REPLAY=1 (profiling only): every phase is proven once
// stepwise (k_round per round, host transcript in between: the proof), then
// its input tables are restored and the production kernels run the same
// phase again reading the recorded challenges from device memory
// (RecordedChallenges).  Under ncu the second run is what to capture
// (-k regex:"k_sumcheck_(persistent|cluster)"): the persistent / cluster
// kernels, replayable, with no host in the loop.  Their folded tables are
// compared with the stepwise run's so a replay that diverged is an error.
template <class F>
static int run_phase_replay(PhaseArgs<F>& a, HostTranscript& tr, uint8_t* rounds_out,
                            uint8_t* point_out, typename F::T* finals_out, cudaStream_t s) {
  using T = typename F::T;
  constexpr int nb = F::kBytes;
  const int n = a.num_vars, k = a.k;
  if (a.prepare) {  // lazily computed round constants: no replay, prove as usual
    a.replaying = true;
    int rc = run_phase_stepwise<F>(a, tr, rounds_out, point_out, finals_out, s);
    a.replaying = false;
    return rc;
  }
  const size_t bytes = ((size_t)1 << n) * sizeof(T);
  std::vector<void*> saved(k, nullptr);
  for (int q = 0; q < k; q++) {
    ZKL_CUDA(cudaMalloc(&saved[q], bytes));
    ZKL_CUDA(cudaMemcpyAsync(saved[q], a.tables[q], bytes, cudaMemcpyDeviceToDevice, s));
  }
  std::vector<T> fin(k);
  int rc = run_phase_stepwise<F>(a, tr, rounds_out, point_out, fin.data(), s);
  if (finals_out)
    for (int q = 0; q < k; q++) finals_out[q] = fin[q];
  std::vector<uint32_t> words((size_t)n * (nb / 4));
  for (int j = 0; j < n && !rc; j++) {
    const T r = host::from_canon<F>(point_out + (size_t)j * nb);
    memcpy(words.data() + (size_t)j * (nb / 4), &r, nb);
  }
  void* dw = nullptr;
  if (!rc) {
    ZKL_CUDA(cudaMalloc(&dw, words.size() * 4));
    ZKL_CUDA(cudaMemcpyAsync(dw, words.data(), words.size() * 4, cudaMemcpyHostToDevice, s));
    for (int q = 0; q < k; q++)
      ZKL_CUDA(cudaMemcpyAsync(a.tables[q], saved[q], bytes, cudaMemcpyDeviceToDevice, s));
    HostTranscript scratch = tr;  // the replay appends nothing: the host loop is skipped
    a.replaying = true;
    a.replay_words = dw;
    rc = run_phase<F>(a, scratch, rounds_out, point_out, nullptr, s);
    a.replaying = false;
    a.replay_words = nullptr;
    a.stepwise = true;  // finals come from the stepwise run (fin_cache)
  }
  if (!rc) {  // the replay must end on the stepwise run's folded values
    for (int q = 0; q < k; q++) {
      T v[2];
      ZKL_CUDA(cudaMemcpyAsync(v, a.tables[q], 2 * sizeof(T), cudaMemcpyDeviceToHost, s));
      ZKL_CUDA(cudaStreamSynchronize(s));
      using H = typename host::For<F>::H;
      const T r = host::from_canon<F>(point_out + (size_t)(n - 1) * nb);
      const T f = H::add(v[0], H::mul(r, H::sub(v[1], v[0])));
      if (memcmp(&f, &fin[q], sizeof(T)) != 0) {
        set_error("profile replay: the production kernels diverged from the stepwise proof "
                  "(table %d of %d, %d rounds, shape %d)", q, k, n,
                  a.forced_shape >= 0 ? a.forced_shape : detect_shape<F>(a.tm));
        rc = kErrArg;
      }
    }
  }
  for (void* p : saved) cudaFree(p);
  if (dw) cudaFree(dw);
  return rc;
}

template <class F>
int op_sumcheck_prove(void* const* tables, int k, int num_vars, const Terms<F>& tm,
                      const typename F::T* post_add, const typename F::T& post_mul,
                      uint8_t* state, uint8_t* rounds_out, uint8_t* point_out,
                      uint8_t* finals_out, cudaStream_t s) {
  using T = typename F::T;
  const int nb = F::kBytes;
  if (k < 1 || k > kMaxTables || tm.nterms < 0 || tm.nterms > kMaxTerms || tm.degree < 0 ||
      tm.degree > 3) {
    set_error("sumcheck_prove: bad arguments");
    return kErrArg;
  }
  if (num_vars == 0) return kOk;
  // ZKL_NO_PERSISTENT=1: one launch per round.  Also chosen automatically
  // under tools that inject into the process and serialise / replay kernels
  // (ncu, compute-sanitizer): a replayed kernel
  // would spin on a mailbox the host never answers.
  HostTranscript tr;
  memcpy(tr.state, state, 64);
  if (no_persistent() && !profile_replay()) {
    uint64_t size = 1ull << num_vars;
    T r_prev = F::zero();
    for (int j = 0; j < num_vars; j++) {
      Post<F> post;
      post.add = post_add ? post_add[j] : F::zero();
      post.mul = post_mul;
      uint8_t* rj = rounds_out + (size_t)j * (tm.degree + 1) * nb;
      int rc = op_sumcheck_round<F>(tables, k, size, j > 0, r_prev, tm, post, rj, s);
      if (rc) return rc;
      if (j > 0) size >>= 1;
      for (int x = 0; x <= tm.degree; x++) tr.append_elem("sumcheck/eval", rj + x * nb, nb);
      challenge_canon<F>(tr, "sumcheck/round", point_out + (size_t)j * nb);
      r_prev = load_canon<F>(point_out + (size_t)j * nb);
    }
    memcpy(state, tr.state, 64);
    return op_sumcheck_finish<F>(tables, k, r_prev, finals_out, s);
  }
  PhaseArgs<F> a;
  a.tables = tables;
  a.k = k;
  a.num_vars = num_vars;
  a.tm = tm;
  a.post_add = post_add;
  a.post_mul = post_mul;
  a.host_tail = host_tail_default();
  std::vector<T> fin(k);
  int rc = run_phase<F>(a, tr, rounds_out, point_out, fin.data(), s);
  if (rc) return rc;
  for (int q = 0; q < k; q++) host::to_canon<F>(finals_out + (size_t)q * nb, fin[q]);
  memcpy(state, tr.state, 64);
  return kOk;
}

// The replicated logUp claim's first `rounds` rounds (the high log2(d/n)
// variables) with the eq-factored tiled evaluator (EvLogupTiled), then A, S
// folded by the last challenge and the eq table of the remaining tile_log
// variables (E folded at the bound point) written to tables[0], ready for
// the next phase over 2^tile_log-entry tables.
// tables: [E_out (2^tile_log, written), A, S+beta (2^num_vars, folded in
// place), B, T+beta, M (2^tile_log)]; u: the eq point (num_vars, storage
// form); coefs: the five Eq.-7 term coefficients (storage form);
// flags: 1 = A is 1/S entrywise (the prover's construction); 2 = indexed:
// tables[6] is the uint32 query -> table index, A = B[index], S = T[index]
// are never materialised, and tables[1], tables[2] are 2^(num_vars-1)-entry
// outputs that the first fold writes.
template <class F>
int op_logup_tiled(void* const* tables, int tile_log, int num_vars, int rounds,
                   const typename F::T* u, const typename F::T* coefs, int flags,
                   uint8_t* state, uint8_t* rounds_out, uint8_t* point_out, cudaStream_t s) {
  using T = typename F::T;
  using H = typename host::For<F>::H;
  if ((flags & 2) && rounds < 2) {
    set_error("logup_tiled: the indexed mode needs at least two tiled rounds");
    return kErrArg;
  }
  if (no_persistent()) {
    set_error("logup_tiled: needs the persistent engine (stepwise mode active)");
    return kErrUnsupported;
  }
  if (rounds < 1 || rounds > 40 || tile_log < 1 || rounds + tile_log != num_vars) {
    set_error("logup_tiled: bad rounds/tile sizes");
    return kErrArg;
  }
  if (tile_log < 5) {
    set_error("logup_tiled: table side below 32 entries");
    return kErrUnsupported;
  }
  const uint64_t ntile = 1ull << tile_log;
  // the eq_lo-weighted S column needs eq_lo(t) != 0: no tile coordinate of u
  // may be 0 or 1 (a challenge equal to either has probability ~2^-254; the
  // caller then takes the materialised path)
  for (int j = rounds; j < num_vars; j++) {
    if (H::is_zero(u[j]) || H::is_zero(H::sub(u[j], H::one()))) {
      set_error("logup_tiled: eq point coordinate 0 or 1 on the tile variables");
      return kErrUnsupported;
    }
  }
  // eq_hi for every round: round j uses eq(u_{j+1..rounds-1}, k) over
  // 2^(rounds-1-j) entries at offset 2^(rounds-1-j) - 1 (MSB-first, like
  // mle.eq_table); built on the host (2^rounds - 1 entries)
  const size_t nhi = ((size_t)1 << rounds) - 1;
  std::vector<T> hi(nhi);
  for (int j = 0; j < rounds; j++) {
    const int m = rounds - 1 - j;
    T* t = hi.data() + (((size_t)1 << m) - 1);
    t[0] = H::one();
    for (int c = 0; c < m; c++) {  // append coordinate u_{j+1+c} as the new low bit
      const T uc = u[j + 1 + c], vc = H::sub(H::one(), uc);
      for (int64_t q = ((int64_t)1 << c) - 1; q >= 0; q--) {
        t[2 * q + 1] = H::mul(t[q], uc);
        t[2 * q] = H::mul(t[q], vc);
      }
    }
  }
  // the work arena, not scratch: run_phase keeps its block partials in scratch
  void* ws;
  int rc = work_reserve(nhi * sizeof(T) + 2 * ntile * sizeof(T) + 2 * sizeof(T), &ws, s);
  if (rc) return rc;
  T* d_hi = (T*)ws;
  T* d_bt = d_hi + nhi;
  T* d_dot = d_bt + ntile;
  T* d_inv_lo = d_dot + 2;  // 1 / eq_lo, for un-weighting S after the phase
  ZKL_CUDA(cudaMemcpyAsync(d_hi, hi.data(), nhi * sizeof(T), cudaMemcpyHostToDevice, s));
  // eq_lo = eq(u_rounds.., ti) into the E_out buffer; table-side constants
  T* eq_lo = (T*)tables[0];
  if ((rc = op_eq_table<F>(eq_lo, u + rounds, tile_log, s))) return rc;
  if ((rc = op_mul<F>(d_bt, tables[3], tables[4], ntile, s))) return rc;
  if ((rc = op_dot<F>(d_dot, d_bt, eq_lo, ntile, s))) return rc;
  if ((rc = op_dot<F>(d_dot + 1, tables[5], tables[3], ntile, s))) return rc;
  T consts[2];
  ZKL_CUDA(cudaMemcpyAsync(consts, d_dot, 2 * sizeof(T), cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  Terms<F> tm;
  memset(&tm, 0, sizeof(tm));
  tm.nterms = 5;
  tm.degree = 3;
  for (int t = 0; t < 5; t++) tm.coef[t] = coefs[t];
  tm.tile_log = tile_log;
  tm.inv_pair = (flags & 1) ? 1 : 0;
  tm.tiled_d = 1ull << num_vars;
  if (flags & 2) {  // indexed: tables[6] = query -> table index, A / S written from round 1
    tm.sidx = (const uint32_t*)tables[6];
    tm.side_a = (const T*)tables[3];
    tm.side_s = (const T*)tables[4];
    tm.sidx_d = 1ull << num_vars;
  }
  void* phase_tables[4] = {d_hi, tables[1], tables[2], eq_lo};
  HostTranscript tr;
  memcpy(tr.state, state, 64);
  PhaseArgs<F> a;
  a.tables = phase_tables;
  a.k = 4;
  a.num_vars = num_vars;
  a.tm = tm;
  a.post_mul = H::one();
  a.rounds_limit = rounds;
  a.forced_shape = kLogupTiled;
  a.lq_u = u;
  a.lq_k3 = consts[0];
  a.lq_smb = consts[1];
  rc = run_phase<F>(a, tr, rounds_out, point_out, nullptr, s);
  if (rc) return rc;
  const T r = host::from_canon<F>(point_out + (size_t)(rounds - 1) * F::kBytes);
  const uint64_t half = 1ull << (num_vars - rounds);
  for (int j = 1; j < 3; j++)
    if ((rc = op_fold<F>(tables[j], tables[j], half, r, s))) return rc;
  // S was carried weighted by eq_lo (EvLogupTiled) from the first fold on (so
  // only when the phase folded at all): divide the n survivors by it (eq_lo
  // has no zero entry: checked before the phase)
  if (rounds >= 2) {
    int64_t z = -1;
    if ((rc = op_batch_inverse<F>(d_inv_lo, eq_lo, ntile, H::zero(), false, &z, s))) return rc;
    if ((rc = op_mul<F>(tables[2], tables[2], d_inv_lo, ntile, s))) return rc;
  }
  // E at the bound point: C * eq_lo with C = prod_j ((1 - u_j) + r_j (2 u_j - 1))
  T c = H::one();
  for (int j = 0; j < rounds; j++) {
    const T rj = host::from_canon<F>(point_out + (size_t)j * F::kBytes);
    const T uj = u[j];
    c = H::mul(c, H::add(H::sub(H::one(), uj), H::mul(rj, H::sub(H::add(uj, uj), H::one()))));
  }
  if ((rc = op_axpy<F>(eq_lo, eq_lo, H::sub(c, H::one()), eq_lo, ntile, s))) return rc;
  memcpy(state, tr.state, 64);
  return kOk;
}

#define ZKL_INST_PERSIST(F)                                                                   \
  template int op_logup_tiled<F>(void* const*, int, int, int, const F::T*, const F::T*, int,  \
                                 uint8_t*, uint8_t*, uint8_t*, cudaStream_t);                 \
  template int detect_shape<F>(const Terms<F>&);                                              \
  template int run_phase<F>(PhaseArgs<F>&, HostTranscript&, uint8_t*, uint8_t*, F::T*,         \
                            cudaStream_t);                                                    \
  template int wait_phase_finals<F>(const PhaseArgs<F>&, F::T*, cudaStream_t);                \
  template int op_sumcheck_prove<F>(void* const*, int, int, const Terms<F>&, const F::T*,     \
                                    const F::T&, uint8_t*, uint8_t*, uint8_t*, uint8_t*,      \
                                    cudaStream_t);
ZKL_INST_PERSIST(Fr255)
ZKL_INST_PERSIST(M61)

}  // namespace zkl
