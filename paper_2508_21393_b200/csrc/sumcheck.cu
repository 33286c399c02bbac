// Dense product sumcheck: fused fold(previous challenge) + round evaluation.
//
// Reference: sumcheck.py:98-130 (prove_sumcheck).  One call = one round:
//   if fold: t[j][i] <- t[j][i] + r_prev (t[j][i + S/2] - t[j][i]) for the
//            whole table (S = current size), in place, fused with
//   evals[x] = post_mul * (post_add + sum_{i < half} combine(terms, t_x(i)))
//            for x = 0..degree, t_x = (1-x) t[i] + x t[i+half] (g(1) is
//            computed directly, never derived from the claim).
// The per-block partial sums are reduced by the last block to finish
// (threadfence + ticket), which converts to canonical form; one D2H copy.
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

template <class F>
struct RoundOut {
  typename F::T* partials;  // gridDim.x * 4
  unsigned* ticket;
  typename F::T* evals_canon;  // 4 (canonical)
};

template <class F, int MAXK, bool FOLD>
__global__ void __launch_bounds__(256) k_round(TablePtrs<F, MAXK> tabs, int k, uint64_t half,
                                               typename F::T r, Terms<F> tm, Post<F> post,
                                               RoundOut<F> out) {
  using T = typename F::T;
  __shared__ T sm[8 * 4];
  __shared__ bool last;
  T acc[4] = {F::zero(), F::zero(), F::zero(), F::zero()};
  const int deg = tm.degree;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < half;
       i += (uint64_t)gridDim.x * blockDim.x) {
    T cur[MAXK], df[MAXK];
#pragma unroll
    for (int j = 0; j < MAXK; j++) {
      if (j < k) {
        T* t = tabs.t[j];
        T lo, hi;
        if (FOLD) {
          T a0 = t[i], a1 = t[i + 2 * half], b0 = t[i + half], b1 = t[i + 3 * half];
          lo = F::add(a0, F::mul(r, F::sub(a1, a0)));
          hi = F::add(b0, F::mul(r, F::sub(b1, b0)));
          t[i] = lo;
          t[i + half] = hi;
        } else {
          lo = t[i];
          hi = t[i + half];
        }
        cur[j] = lo;
        df[j] = F::sub(hi, lo);
      } else {
        cur[j] = F::zero();
        df[j] = F::zero();
      }
    }
    acc[0] = F::add(acc[0], combine_terms<F, MAXK>(cur, tm));
#pragma unroll
    for (int x = 1; x < 4; x++) {
      if (x <= deg) {
#pragma unroll
        for (int j = 0; j < MAXK; j++)
          if (j < k) cur[j] = F::add(cur[j], df[j]);
        acc[x] = F::add(acc[x], combine_terms<F, MAXK>(cur, tm));
      }
    }
  }
  block_sum<F, 4>(acc, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int x = 0; x < 4; x++) out.partials[blockIdx.x * 4 + x] = acc[x];
    __threadfence();
    unsigned tk = atomicAdd(out.ticket, 1u);
    last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  // last block: reduce all partials
  __threadfence();
  T v[4] = {F::zero(), F::zero(), F::zero(), F::zero()};
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int x = 0; x < 4; x++) v[x] = F::add(v[x], ld_cg(out.partials + b * 4 + x));
  }
  block_sum<F, 4>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int x = 0; x < 4; x++)
      out.evals_canon[x] = F::from_mont(F::mul(post.mul, F::add(v[x], post.add)));
    *out.ticket = 0;  // reset for the next launch
  }
}

template <class F, int MAXK>
static int launch_round(void* const* tables, int k, uint64_t half, bool fold,
                        typename F::T r, const Terms<F>& tm, const Post<F>& post,
                        RoundOut<F> out, unsigned grid, cudaStream_t s) {
  TablePtrs<F, MAXK> tp;
  for (int j = 0; j < MAXK; j++) tp.t[j] = j < k ? (typename F::T*)tables[j] : nullptr;
  if (fold)
    k_round<F, MAXK, true><<<grid, 256, 0, s>>>(tp, k, half, r, tm, post, out);
  else
    k_round<F, MAXK, false><<<grid, 256, 0, s>>>(tp, k, half, r, tm, post, out);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

template <class F>
int op_sumcheck_round(void* const* tables, int k, uint64_t size, bool fold,
                      typename F::T r_prev, const Terms<F>& tm, const Post<F>& post,
                      uint8_t* evals_host, cudaStream_t s) {
  using T = typename F::T;
  if (k < 1 || k > kMaxTables) { set_error("sumcheck: %d tables unsupported", k); return kErrArg; }
  if (tm.nterms < 0 || tm.nterms > kMaxTerms || tm.degree < 0 || tm.degree > 3) {
    set_error("sumcheck: bad terms/degree");
    return kErrArg;
  }
  // pairs evaluated this round
  uint64_t half = fold ? size / 4 : size / 2;
  if (half == 0) { set_error("sumcheck: table too small for a round"); return kErrArg; }
  unsigned grid = grid_for(half, 256, k > 4 ? 2 : 4);
  void* ws;
  size_t need = (size_t)grid * 4 * sizeof(T) + 4 * sizeof(T) + 64;
  int rc = scratch_reserve(need, &ws, s);
  if (rc) return rc;
  RoundOut<F> out;
  out.partials = (T*)ws;
  out.evals_canon = out.partials + (size_t)grid * 4;
  out.ticket = (unsigned*)(out.evals_canon + 4);
  ZKL_CUDA(cudaMemsetAsync(out.ticket, 0, sizeof(unsigned), s));
  if (k <= 2)
    rc = launch_round<F, 2>(tables, k, half, fold, r_prev, tm, post, out, grid, s);
  else if (k <= 4)
    rc = launch_round<F, 4>(tables, k, half, fold, r_prev, tm, post, out, grid, s);
  else
    rc = launch_round<F, 8>(tables, k, half, fold, r_prev, tm, post, out, grid, s);
  if (rc) return rc;
  void* pin;
  rc = pinned_reserve(4 * sizeof(T), &pin);
  if (rc) return rc;
  ZKL_CUDA(cudaMemcpyAsync(pin, out.evals_canon, 4 * sizeof(T), cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  memcpy(evals_host, pin, (size_t)(tm.degree + 1) * sizeof(T));
  return kOk;
}

template <class F, int MAXK>
__global__ void k_finish(TablePtrs<F, MAXK> tabs, int k, typename F::T r,
                         typename F::T* out_canon) {
  int j = threadIdx.x;
  if (j < k) {
    typename F::T a = tabs.t[j][0], b = tabs.t[j][1];
    out_canon[j] = F::from_mont(F::add(a, F::mul(r, F::sub(b, a))));
  }
}

template <class F>
int op_sumcheck_finish(void* const* tables, int k, typename F::T r, uint8_t* finals_host,
                       cudaStream_t s) {
  using T = typename F::T;
  if (k < 1 || k > kMaxTables) { set_error("finish: bad k"); return kErrArg; }
  void* ws;
  int rc = scratch_reserve(kMaxTables * sizeof(T), &ws, s);
  if (rc) return rc;
  TablePtrs<F, kMaxTables> tp;
  for (int j = 0; j < kMaxTables; j++) tp.t[j] = j < k ? (T*)tables[j] : nullptr;
  k_finish<F, kMaxTables><<<1, 32, 0, s>>>(tp, k, r, (T*)ws);
  ZKL_LAUNCH_CHECK();
  void* pin;
  rc = pinned_reserve(kMaxTables * sizeof(T), &pin);
  if (rc) return rc;
  ZKL_CUDA(cudaMemcpyAsync(pin, ws, k * sizeof(T), cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  memcpy(finals_host, pin, k * sizeof(T));
  return kOk;
}

#define ZKL_INST_SC(F)                                                                  \
  template int op_sumcheck_round<F>(void* const*, int, uint64_t, bool, F::T,            \
                                    const Terms<F>&, const Post<F>&, uint8_t*,          \
                                    cudaStream_t);                                      \
  template int op_sumcheck_finish<F>(void* const*, int, F::T, uint8_t*, cudaStream_t);
ZKL_INST_SC(Fr255)
ZKL_INST_SC(M61)

}  // namespace zkl
