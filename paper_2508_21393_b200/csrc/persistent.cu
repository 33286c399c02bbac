// Persistent whole-sumcheck driver (sumcheck.py:108-130 after _absorb_claim).
//
// ONE cooperative launch runs every round.  Per round:
//   1. every thread folds its pairs by the previous challenge (in place) and
//      accumulates shape-specific raw sums (no term coefficients on device);
//   2. warp shuffles reduce them; lane 0 of every warp writes a partial;
//   3. grid barrier; warp 0 of block 0 sums the partials and publishes the raw
//      sums (Montgomery form) into a mailbox in mapped pinned host memory;
//   4. the host applies the term coefficients / post-scalars, converts to
//      canonical form, runs the native SHAKE-256 transcript (transcript.cu)
//      and writes the next challenge back; block 0 spins on it (PCIe);
//   5. grid barrier; every block picks up the challenge.
// No kernel launches, copies or stream syncs per round.  Scalar field work
// sits on the host because a dependent Montgomery multiply costs ~1.6k
// cycles on one GPU thread (scratch/lat.cu) but ~0.1 us on the host.
//
// Shapes (detected from the term list on the host):
//   GENERIC  : any terms; device applies coefficients (combine, sumcheck.py:70)
//   PROD2    : c * t_a t_b          -- zkMat U/W phases; 3 mults per pair
//   PROD3    : c * t_a t_b t_c      -- elementprod; 7 mults per pair
//   SUM2PROD2: c0 t_a t_b + c1 t_a t_c -- zkMat V phase; 6 mults per pair
// The quadratic products use p(2) = 2p(1) - p(0) + 2c, p(3) = 3p(1) - 2p(0) + 6c
// with c = (t_a(1)-t_a(0))(t_b(1)-t_b(0)): every evaluation is still computed
// from the tables, never derived from the claimed sum.
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <vector>

#include <cooperative_groups.h>

#include "round_eval.cuh"
#include "transcript.cuh"

namespace cg = cooperative_groups;

namespace zkl {

enum Shape { kGeneric = 0, kProd2 = 1, kProd3 = 2, kSum2Prod2 = 3 };

// ---------------------------------------------------------------------------
// evaluators: pair() accumulates, finish() -> NOUT raw sums (4 per group)
template <class F, int MAXK>
struct EvGeneric {
  using T = typename F::T;
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
};

// quadratic-product helper: (c0, c1, c2) -> p(0..3)
template <class F>
ZKL_D void quad_evals(const typename F::T& c0, const typename F::T& c1, const typename F::T& c2,
                      typename F::T* out) {
  using T = typename F::T;
  const T two_c1 = F::add(c1, c1), two_c2 = F::add(c2, c2);
  out[0] = c0;
  out[1] = c1;
  out[2] = F::sub(F::add(two_c1, two_c2), c0);                      // 2c1 - c0 + 2c2
  const T six_c2 = F::add(F::add(two_c2, two_c2), two_c2);
  out[3] = F::sub(F::add(F::add(two_c1, c1), six_c2), F::add(c0, c0));  // 3c1 - 2c0 + 6c2
}

template <class F, int MAXK>
struct EvProd2 {
  using T = typename F::T;
  static constexpr int NA = 3, NOUT = 4;
  ZKL_D static void pair(T (&cur)[MAXK], const T (&df)[MAXK], int, const Terms<F>& tm,
                         T (&acc)[NA]) {
    const int a = tm.fi[0][0], b = tm.fi[0][1];
    const T f0 = select_tab<F, MAXK>(cur, a), fd = select_tab<F, MAXK>(df, a);
    const T g0 = select_tab<F, MAXK>(cur, b), gd = select_tab<F, MAXK>(df, b);
    T p0, pc;
    F::mul2(f0, g0, fd, gd, p0, pc);
    const T p1 = F::mul(F::add(f0, fd), F::add(g0, gd));
    acc[0] = F::add(acc[0], p0);
    acc[1] = F::add(acc[1], p1);
    acc[2] = F::add(acc[2], pc);
  }
  ZKL_D static void finish(const T (&acc)[NA], T (&out)[NOUT]) {
    quad_evals<F>(acc[0], acc[1], acc[2], out);
  }
};

template <class F, int MAXK>
struct EvSum2Prod2 {
  using T = typename F::T;
  static constexpr int NA = 6, NOUT = 8;
  ZKL_D static void pair(T (&cur)[MAXK], const T (&df)[MAXK], int, const Terms<F>& tm,
                         T (&acc)[NA]) {
    const int a = tm.fi[0][0], b = tm.fi[0][1], c = tm.fi[1][1];
    const T f0 = select_tab<F, MAXK>(cur, a), fd = select_tab<F, MAXK>(df, a);
    const T g0 = select_tab<F, MAXK>(cur, b), gd = select_tab<F, MAXK>(df, b);
    const T h0 = select_tab<F, MAXK>(cur, c), hd = select_tab<F, MAXK>(df, c);
    const T f1 = F::add(f0, fd);
    T m[6];
    F::mul2(f0, g0, f0, h0, m[0], m[3]);
    F::mul2(f1, F::add(g0, gd), f1, F::add(h0, hd), m[1], m[4]);
    F::mul2(fd, gd, fd, hd, m[2], m[5]);
#pragma unroll
    for (int q = 0; q < 6; q++) acc[q] = F::add(acc[q], m[q]);
  }
  ZKL_D static void finish(const T (&acc)[NA], T (&out)[NOUT]) {
    quad_evals<F>(acc[0], acc[1], acc[2], out);
    quad_evals<F>(acc[3], acc[4], acc[5], out + 4);
  }
};

template <class F, int MAXK>
struct EvProd3 {
  using T = typename F::T;
  static constexpr int NA = 4, NOUT = 4;
  ZKL_D static void pair(T (&cur)[MAXK], const T (&df)[MAXK], int, const Terms<F>& tm,
                         T (&acc)[NA]) {
    const int a = tm.fi[0][0], b = tm.fi[0][1], c = tm.fi[0][2];
    const T e0 = select_tab<F, MAXK>(cur, a), ed = select_tab<F, MAXK>(df, a);
    const T a0 = select_tab<F, MAXK>(cur, b), ad = select_tab<F, MAXK>(df, b);
    const T b0 = select_tab<F, MAXK>(cur, c), bd = select_tab<F, MAXK>(df, c);
    T q[4], q0, qc;
    F::mul2(e0, a0, ed, ad, q0, qc);
    quad_evals<F>(q0, F::mul(F::add(e0, ed), F::add(a0, ad)), qc, q);
    const T b1 = F::add(b0, bd), b2 = F::add(b1, bd), b3 = F::add(b2, bd);
    T m[4];
    F::mul2(q[0], b0, q[1], b1, m[0], m[1]);
    F::mul2(q[2], b2, q[3], b3, m[2], m[3]);
#pragma unroll
    for (int x = 0; x < 4; x++) acc[x] = F::add(acc[x], m[x]);
  }
  ZKL_D static void finish(const T (&acc)[NA], T (&out)[NOUT]) {
#pragma unroll
    for (int x = 0; x < 4; x++) out[x] = acc[x];
  }
};

// ---------------------------------------------------------------------------
// mailbox access (host-mapped memory: every device read is a PCIe round trip)
ZKL_D uint32_t ld_acquire_sys(const volatile uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
ZKL_D void st_release_sys(volatile uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
ZKL_D void st_vec_sys(volatile uint8_t* dst, const void* src, int nbytes) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  for (int o = 0; o < nbytes; o += 16) {
    uint4 v = s[o / 16];
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(dst + o), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  }
}
ZKL_D void ld_vec32_sys(void* dst, const volatile uint8_t* src) {
  uint4 v0, v1;  // both loads in flight together
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v0.x), "=r"(v0.y), "=r"(v0.z), "=r"(v0.w)
               : "l"(src)
               : "memory");
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v1.x), "=r"(v1.y), "=r"(v1.z), "=r"(v1.w)
               : "l"(src + 16)
               : "memory");
  reinterpret_cast<uint4*>(dst)[0] = v0;
  reinterpret_cast<uint4*>(dst)[1] = v1;
}
ZKL_D uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr uint64_t kSpinTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s

template <class F, int MAXK, class EV>
__global__ void __launch_bounds__(256)
    k_sumcheck_persistent(TablePtrs<F, MAXK> tabs, int k, int num_vars, Terms<F> tm,
                          Mailbox* mb, typename F::T* partials, typename F::T* rbuf,
                          unsigned* fail, uint64_t* trace) {
  using T = typename F::T;
  cg::grid_group g = cg::this_grid();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  __shared__ T wsum[8 * EV::NOUT];
  uint64_t size = 1ull << num_vars;
  T r = F::zero();
  const bool tr0 = trace && blockIdx.x == 0 && threadIdx.x == 0;
  for (int j = 0; j < num_vars; j++) {
    if (tr0) trace[j * 6 + 0] = globaltimer();
    const bool fold = j > 0;
    const uint64_t half = fold ? size >> 2 : size >> 1;
    T acc[EV::NA];
#pragma unroll
    for (int q = 0; q < EV::NA; q++) acc[q] = F::zero();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < half;
         i += (uint64_t)gridDim.x * blockDim.x) {
      T cur[MAXK], df[MAXK];
      if (fold)
        load_pair<F, MAXK, true, true>(tabs, k, i, half, r, cur, df);
      else
        load_pair<F, MAXK, false, true>(tabs, k, i, half, r, cur, df);
      EV::pair(cur, df, k, tm, acc);
    }
    T out[EV::NOUT];
    EV::finish(acc, out);
#pragma unroll
    for (int q = 0; q < EV::NOUT; q++) out[q] = warp_sum<F>(out[q]);
    // block partial: warp sums -> shared -> warp 0 (one partial per block)
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < EV::NOUT; q++) wsum[warp * EV::NOUT + q] = out[q];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < EV::NOUT; q++) {
        T s = lane < nwarps ? wsum[lane * EV::NOUT + q] : F::zero();
        s = warp_sum<F>(s);
        if (lane == 0) partials[(size_t)blockIdx.x * EV::NOUT + q] = s;
      }
    }
    if (tr0) trace[j * 6 + 1] = globaltimer();
    g.sync();
    if (tr0) trace[j * 6 + 2] = globaltimer();
    if (blockIdx.x == 0 && warp == 0) {
      T v[EV::NOUT];
#pragma unroll
      for (int q = 0; q < EV::NOUT; q++) v[q] = F::zero();
      for (unsigned w = lane; w < gridDim.x; w += 32) {
#pragma unroll
        for (int q = 0; q < EV::NOUT; q++)
          v[q] = F::add(v[q], ld_cg(partials + (size_t)w * EV::NOUT + q));
      }
#pragma unroll
      for (int q = 0; q < EV::NOUT; q++) v[q] = warp_sum<F>(v[q]);
      if (lane == 0) {
        alignas(16) T pub[EV::NOUT];
#pragma unroll
        for (int q = 0; q < EV::NOUT; q++) pub[q] = v[q];
        st_vec_sys(mb->evals, pub, (int)sizeof(pub));
        __threadfence_system();
        st_release_sys(&mb->ev_seq, (uint32_t)(j + 1));
        if (tr0) trace[j * 6 + 3] = globaltimer();
        const uint64_t t0 = globaltimer();
        unsigned bad = 0;
        for (uint32_t spin = 1; ld_acquire_sys(&mb->ch_seq) != (uint32_t)(j + 1); spin++) {
          if ((spin & 63) == 0 &&
              (ld_acquire_sys(&mb->abort) || globaltimer() - t0 > kSpinTimeoutNs)) {
            bad = 1;
            break;
          }
        }
        if (bad) {
          *fail = 1;
          mb->status = 1;
        } else {
          alignas(16) uint8_t cb[32];
          ld_vec32_sys(cb, mb->chal);
          T c;
          memcpy(&c, cb, F::kBytes);
          *rbuf = c;
        }
        if (tr0) trace[j * 6 + 4] = globaltimer();
        __threadfence();
      }
    }
    g.sync();
    if (tr0) trace[j * 6 + 5] = globaltimer();
    if (ld_cg(fail)) return;
    r = ld_cg(rbuf);
    if (fold) size >>= 1;
  }
  // final fold of the size-2 tables by the last challenge (sumcheck.py:129-130)
  if (blockIdx.x == 0) {
    __shared__ T fin[MAXK];
    if (threadIdx.x < k) {
      const T* t = tabs.t[threadIdx.x];
      T a = ld_cg(t), b = ld_cg(t + 1);
      fin[threadIdx.x] = F::from_mont(F::add(a, F::mul(r, F::sub(b, a))));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      alignas(16) T buf[MAXK];
      for (int q = 0; q < k; q++) buf[q] = fin[q];
      st_vec_sys(mb->finals, buf, (k * F::kBytes + 15) & ~15);
      __threadfence_system();
    }
  }
}

// ---------------------------------------------------------------------------
template <class F, int MAXK, class EV>
struct Persistent {
  static int grid(uint64_t half0) {
    static int per_sm = -1;
    if (per_sm < 0) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
              &per_sm, k_sumcheck_persistent<F, MAXK, EV>, 256, 0) != cudaSuccess ||
          per_sm < 1)
        per_sm = 1;
    }
    int dev = 0, sms = kSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t cap = (uint64_t)sms * per_sm;
    uint64_t want = (half0 + 255) / 256;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
  }
  static int launch(void* const* tables, int k, int num_vars, const Terms<F>& tm, Mailbox* mb,
                    typename F::T* partials, typename F::T* rbuf, unsigned* fail,
                    uint64_t* trace, unsigned grid, cudaStream_t s) {
    TablePtrs<F, MAXK> tp;
    for (int j = 0; j < MAXK; j++) tp.t[j] = j < k ? (typename F::T*)tables[j] : nullptr;
    Terms<F> tmc = tm;
    void* args[] = {&tp, &k, &num_vars, &tmc, &mb, &partials, &rbuf, &fail, &trace};
    ZKL_CUDA(cudaLaunchCooperativeKernel((const void*)k_sumcheck_persistent<F, MAXK, EV>, grid,
                                         256, args, 0, s));
    ZKL_LAUNCH_CHECK();
    return kOk;
  }
};

template <class F>
static int detect_shape(const Terms<F>& tm) {
  if (tm.nterms == 1 && tm.nf[0] == 2) return kProd2;
  if (tm.nterms == 1 && tm.nf[0] == 3) return kProd3;
  if (tm.nterms == 2 && tm.nf[0] == 2 && tm.nf[1] == 2 && tm.fi[0][0] == tm.fi[1][0])
    return kSum2Prod2;
  return kGeneric;
}

template <class F, int MAXK>
static int dispatch(int shape, bool query, uint64_t half0, int* grid_out, void* const* tables,
                    int k, int num_vars, const Terms<F>& tm, Mailbox* mb, typename F::T* partials,
                    typename F::T* rbuf, unsigned* fail, uint64_t* trace, cudaStream_t s,
                    int* nout) {
#define ZKL_SHAPE(EVT)                                                                      \
  {                                                                                         \
    using P = Persistent<F, MAXK, EVT<F, MAXK>>;                                            \
    *nout = EVT<F, MAXK>::NOUT;                                                             \
    if (query) { *grid_out = P::grid(half0); return kOk; }                                  \
    return P::launch(tables, k, num_vars, tm, mb, partials, rbuf, fail, trace,              \
                     (unsigned)*grid_out, s);                                                \
  }
  switch (shape) {
    case kProd2: ZKL_SHAPE(EvProd2)
    case kProd3: ZKL_SHAPE(EvProd3)
    case kSum2Prod2: ZKL_SHAPE(EvSum2Prod2)
    default: ZKL_SHAPE(EvGeneric)
  }
#undef ZKL_SHAPE
}

template <class F>
static int run_dispatch(int shape, bool query, uint64_t half0, int* grid, void* const* tables,
                        int k, int num_vars, const Terms<F>& tm, Mailbox* mb,
                        typename F::T* partials, typename F::T* rbuf, unsigned* fail,
                        uint64_t* trace, cudaStream_t s, int* nout) {
  if (k <= 2)
    return dispatch<F, 2>(shape, query, half0, grid, tables, k, num_vars, tm, mb, partials, rbuf,
                          fail, trace, s, nout);
  if (k <= 4)
    return dispatch<F, 4>(shape, query, half0, grid, tables, k, num_vars, tm, mb, partials, rbuf,
                          fail, trace, s, nout);
  return dispatch<F, 8>(shape, query, half0, grid, tables, k, num_vars, tm, mb, partials, rbuf,
                        fail, trace, s, nout);
}

// host: raw sums (Montgomery) -> canonical evaluations
template <class F>
static void host_evals(int shape, const Terms<F>& tm, const typename F::T* raw,
                       const typename F::T& add, const typename F::T& mul, uint8_t* out) {
  using T = typename F::T;
  for (int x = 0; x <= tm.degree; x++) {
    T v;
    switch (shape) {
      case kProd2:
      case kProd3: v = F::mul(tm.coef[0], raw[x]); break;
      case kSum2Prod2: v = F::add(F::mul(tm.coef[0], raw[x]), F::mul(tm.coef[1], raw[4 + x])); break;
      default: v = raw[x];
    }
    store_canon<F>(out + x * F::kBytes, F::mul(mul, F::add(v, add)));
  }
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
  // (ncu, compute-sanitizer set CUDA_INJECTION64_PATH): a replayed kernel
  // would spin on a mailbox the host never answers.
  static const bool no_persistent =
      getenv("ZKL_NO_PERSISTENT") != nullptr || getenv("CUDA_INJECTION64_PATH") != nullptr ||
      (getenv("CUDA_LAUNCH_BLOCKING") && getenv("CUDA_LAUNCH_BLOCKING")[0] == '1');
  if (no_persistent) {
    HostTranscript tr;
    memcpy(tr.state, state, 64);
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
  Mailbox* mb_host;
  Mailbox* mb_dev;
  int rc = mailbox_for_current_device(&mb_host, &mb_dev);
  if (rc) return rc;
  const int shape = detect_shape<F>(tm);
  const uint64_t half0 = 1ull << (num_vars - 1);
  int grid = 0, nout = 4;
  run_dispatch<F>(shape, true, half0, &grid, tables, k, num_vars, tm, nullptr, nullptr, nullptr,
                  nullptr, nullptr, s, &nout);
  size_t need = (size_t)grid * 8 * 8 * sizeof(T);  // warps x NOUT (<= 8)
  void* ws;
  rc = scratch_reserve(need, &ws, s);
  if (rc) return rc;
  void* fx;
  rc = fixed_words(&fx);
  if (rc) return rc;
  unsigned* fail = (unsigned*)((char*)fx + kFixedFail);
  T* rbuf = (T*)((char*)fx + kFixedRbuf);
  T* partials = (T*)ws;
  ZKL_CUDA(cudaMemsetAsync(fail, 0, sizeof(unsigned), s));
  mb_host->ev_seq = 0;
  mb_host->ch_seq = 0;
  mb_host->abort = 0;
  mb_host->status = 0;
  std::atomic_thread_fence(std::memory_order_seq_cst);

  static const bool tracing = getenv("ZKL_TRACE") != nullptr;
  uint64_t* trace = nullptr;
  std::vector<double> host_seen(num_vars), host_sent(num_vars);
  if (tracing) ZKL_CUDA(cudaMalloc(&trace, (size_t)num_vars * 6 * 8));
  rc = run_dispatch<F>(shape, false, half0, &grid, tables, k, num_vars, tm, mb_dev, partials,
                       rbuf, fail, trace, s, &nout);
  if (rc) return rc;

  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
  };
  HostTranscript tr;
  memcpy(tr.state, state, 64);
  T raw[8];
  for (int j = 0; j < num_vars; j++) {
    const auto until = std::chrono::steady_clock::now() + std::chrono::seconds(30);
    uint64_t spins = 0;
    while (mb_host->ev_seq != (uint32_t)(j + 1)) {
      if ((++spins & 0xffff) == 0) {
        cudaError_t q = cudaStreamQuery(s);
        if (q != cudaErrorNotReady) {
          set_error("persistent sumcheck ended early at round %d: %s", j,
                    cudaGetErrorString(q == cudaSuccess ? cudaErrorUnknown : q));
          return kErrCuda;
        }
        if (std::chrono::steady_clock::now() > until) {
          mb_host->abort = 1;
          cudaStreamSynchronize(s);
          set_error("persistent sumcheck: device did not publish round %d", j);
          return kErrCuda;
        }
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    if (tracing) host_seen[j] = now_us();
    memcpy(raw, (const void*)mb_host->evals, (size_t)nout * sizeof(T));
    uint8_t* rj = rounds_out + (size_t)j * (tm.degree + 1) * nb;
    host_evals<F>(shape, tm, raw, post_add ? post_add[j] : F::zero(), post_mul, rj);
    for (int x = 0; x <= tm.degree; x++) tr.append_elem("sumcheck/eval", rj + x * nb, nb);
    uint8_t* rc_out = point_out + (size_t)j * nb;
    challenge_canon<F>(tr, "sumcheck/round", rc_out);
    T rm = load_canon<F>(rc_out);  // Montgomery form for the device
    memcpy((void*)mb_host->chal, &rm, nb);
    std::atomic_thread_fence(std::memory_order_seq_cst);
    mb_host->ch_seq = (uint32_t)(j + 1);
    if (tracing) host_sent[j] = now_us();
  }
  ZKL_CUDA(cudaStreamSynchronize(s));
  if (mb_host->status) {
    set_error("persistent sumcheck: device timed out waiting for a challenge");
    return kErrCuda;
  }
  memcpy(finals_out, (const void*)mb_host->finals, (size_t)k * nb);
  memcpy(state, tr.state, 64);
  if (tracing) {
    std::vector<uint64_t> tv((size_t)num_vars * 6);
    cudaMemcpy(tv.data(), trace, tv.size() * 8, cudaMemcpyDeviceToHost);
    cudaFree(trace);
    double acc[6] = {0}, hs = 0;
    for (int j = 0; j < num_vars; j++) {
      for (int q = 1; q < 6; q++) acc[q] += (double)(tv[j * 6 + q] - tv[j * 6 + q - 1]) / 1000.0;
      if (j + 1 < num_vars) acc[0] += (double)(tv[(j + 1) * 6] - tv[j * 6 + 5]) / 1000.0;
      hs += host_sent[j] - host_seen[j];
    }
    fprintf(stderr,
            "[zkl trace] n=%d k=%d shape=%d grid=%d per-round us: accum %.2f | sync1 %.2f | "
            "reduce+publish %.2f | wait-challenge %.2f | sync2 %.2f | loop %.2f | host %.2f\n",
            num_vars, k, shape, grid, acc[1] / num_vars, acc[2] / num_vars, acc[3] / num_vars,
            acc[4] / num_vars, acc[5] / num_vars, acc[0] / num_vars, hs / num_vars);
  }
  return kOk;
}

template int op_sumcheck_prove<Fr255>(void* const*, int, int, const Terms<Fr255>&,
                                      const Fr255::T*, const Fr255::T&, uint8_t*, uint8_t*,
                                      uint8_t*, uint8_t*, cudaStream_t);
template int op_sumcheck_prove<M61>(void* const*, int, int, const Terms<M61>&, const M61::T*,
                                    const M61::T&, uint8_t*, uint8_t*, uint8_t*, uint8_t*,
                                    cudaStream_t);

}  // namespace zkl
