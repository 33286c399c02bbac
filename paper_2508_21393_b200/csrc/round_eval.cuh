// Per-pair work of one dense sumcheck round (sumcheck.py:110-123, 129):
// optionally fold every table by the previous challenge (in place), then add
// combine(terms, t_x) for x = 0..degree into the thread's accumulators.
#pragma once
#include "ops.cuh"

namespace zkl {

template <class F, int MAXK>
struct TablePtrs {
  typename F::T* t[MAXK];
};

template <class F, int MAXK>
ZKL_D typename F::T select_tab(const typename F::T (&cur)[MAXK], int idx) {
  typename F::T v = cur[0];
#pragma unroll
  for (int j = 1; j < MAXK; j++)
    if (idx == j) v = cur[j];
  return v;
}

template <class F, int MAXK>
ZKL_D typename F::T combine_terms(const typename F::T (&cur)[MAXK], const Terms<F>& tm) {
  typename F::T total = F::zero();
#pragma unroll 1
  for (int t = 0; t < tm.nterms; t++) {
    typename F::T prod = tm.coef[t];
    for (int s = 0; s < tm.nf[t]; s++) prod = F::mul(prod, select_tab<F, MAXK>(cur, tm.fi[t][s]));
    total = F::add(total, prod);
  }
  return total;
}

// CG: L2-coherent loads (tables written by other blocks earlier in the same
// persistent launch).
template <class F, bool CG>
ZKL_D typename F::T ld_tab(const typename F::T* p) {
  if constexpr (CG) return ld_cg(p);
  else return *p;
}

// Load (and, if FOLD, fold in place) the pair (i, i + half) of every table:
// cur = low value, df = high - low.
template <class F, int MAXK, bool FOLD, bool CG>
ZKL_D void load_pair(const TablePtrs<F, MAXK>& tabs, int k, uint64_t i, uint64_t half,
                     const typename F::T& r, typename F::T (&cur)[MAXK],
                     typename F::T (&df)[MAXK]) {
  using T = typename F::T;
#pragma unroll
  for (int j = 0; j < MAXK; j++) {
    if (j < k) {
      T* t = tabs.t[j];
      T lo, hi;
      if (FOLD) {
        T a0 = ld_tab<F, CG>(t + i), a1 = ld_tab<F, CG>(t + i + 2 * half);
        T b0 = ld_tab<F, CG>(t + i + half), b1 = ld_tab<F, CG>(t + i + 3 * half);
        T ra, rb;
        F::mul2(r, F::sub(a1, a0), r, F::sub(b1, b0), ra, rb);
        lo = F::add(a0, ra);
        hi = F::add(b0, rb);
        t[i] = lo;
        t[i + half] = hi;
      } else {
        lo = ld_tab<F, CG>(t + i);
        hi = ld_tab<F, CG>(t + i + half);
      }
      cur[j] = lo;
      df[j] = F::sub(hi, lo);
    } else {
      cur[j] = F::zero();
      df[j] = F::zero();
    }
  }
}

template <class F, int MAXK, bool FOLD, bool CG>
ZKL_D void pair_accumulate(const TablePtrs<F, MAXK>& tabs, int k, uint64_t i, uint64_t half,
                           const typename F::T& r, const Terms<F>& tm,
                           typename F::T (&acc)[4]) {
  using T = typename F::T;
  T cur[MAXK], df[MAXK];
  load_pair<F, MAXK, FOLD, CG>(tabs, k, i, half, r, cur, df);
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

}  // namespace zkl
