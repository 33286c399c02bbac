// Dense product sumcheck: fused fold(previous challenge) + round evaluation.
//
// Reference: sumcheck.py:98-130 (prove_sumcheck).  Round j:
//   if j > 0: t[i] <- t[i] + r_{j-1} (t[i + S/2] - t[i]) for every table (in
//             place, S = current size), fused with
//   evals[x] = post_mul * (post_add_j + sum_{i < half} combine(terms, t_x(i)))
//             for x = 0..degree, t_x = (1-x) t[i] + x t[i+half]  (g(1) is
//             computed directly, never derived from the claim).
//
// Two drivers:
//  * op_sumcheck_round: one launch per round (last-block reduction), evals
//    copied back; used when the caller's transcript is a Python object.
//  * op_sumcheck_prove: ONE persistent cooperative launch for the whole
//    sumcheck.  After each round's grid-wide reduction, block 0 publishes the
//    evaluations into a mailbox in mapped pinned host memory and spins until
//    the host (native SHAKE-256 transcript, transcript.cu) writes back the
//    challenge; a grid barrier then releases every block into the fused
//    fold+evaluate of the next round.  No launches, memcpys or stream syncs
//    per round: the round latency is PCIe round trip + 7 Keccak-f on the host.
#include "round_eval.cuh"

namespace zkl {

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
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < half;
       i += (uint64_t)gridDim.x * blockDim.x)
    pair_accumulate<F, MAXK, FOLD, false>(tabs, k, i, half, r, tm, acc);
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
    *out.ticket = 0;  // ready for the next launch
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

static int check_args(int k, int nterms, int degree) {
  if (k < 1 || k > kMaxTables) { set_error("sumcheck: %d tables unsupported", k); return kErrArg; }
  if (nterms < 0 || nterms > kMaxTerms || degree < 0 || degree > 3) {
    set_error("sumcheck: bad terms/degree");
    return kErrArg;
  }
  return kOk;
}

template <class F>
int op_sumcheck_round(void* const* tables, int k, uint64_t size, bool fold,
                      typename F::T r_prev, const Terms<F>& tm, const Post<F>& post,
                      uint8_t* evals_host, cudaStream_t s) {
  using T = typename F::T;
  int rc = check_args(k, tm.nterms, tm.degree);
  if (rc) return rc;
  uint64_t half = fold ? size / 4 : size / 2;
  if (half == 0) { set_error("sumcheck: table too small for a round"); return kErrArg; }
  unsigned grid = grid_for(half, 256, k > 4 ? 2 : 4);
  // scratch: evals | partials; the ticket lives in the fixed words (zeroed
  // once, reset to 0 by the last block of every launch)
  size_t need = 4 * sizeof(T) + (size_t)grid * 4 * sizeof(T);
  void* ws;
  rc = scratch_reserve(need, &ws, s);
  if (rc) return rc;
  void* fx;
  rc = fixed_words(&fx);
  if (rc) return rc;
  RoundOut<F> out;
  out.ticket = (unsigned*)((char*)fx + kFixedTicket);
  out.evals_canon = (T*)ws;
  out.partials = out.evals_canon + 4;
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
  T* out = (T*)ws;
  TablePtrs<F, kMaxTables> tp;
  for (int j = 0; j < kMaxTables; j++) tp.t[j] = j < k ? (T*)tables[j] : nullptr;
  k_finish<F, kMaxTables><<<1, 32, 0, s>>>(tp, k, r, out);
  ZKL_LAUNCH_CHECK();
  void* pin;
  rc = pinned_reserve(kMaxTables * sizeof(T), &pin);
  if (rc) return rc;
  ZKL_CUDA(cudaMemcpyAsync(pin, out, k * sizeof(T), cudaMemcpyDeviceToHost, s));
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
