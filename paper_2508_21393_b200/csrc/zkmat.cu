// Native zkMat driver: the whole sumcheck of prove_matmul in one C call.
//
// Reference: gadgets.py:241-251 -- draw r_u (d0), r_v (d2), absorb the claim
//   sum_{u,w,v} eq(r_u,u) eq(r_v,v) [A(u,w) B(w,v) - 2^-d1 C(u,v)] = 0
// (sumcheck.py:90-95) and run d0+d1+d2 rounds over the four replicated
// tables of gadgets.py:210-227.  The rounds are produced by the factored
// prover, bit-identical, without materialising any table:
//   U (d0 rounds): (E_u, h),  h = A (B E_v) - C E_v
//   W (d1 rounds): E_hat [ sum a bv - 2^-d1 2^(d1-j-1) kappa ],
//                  a = E(rho_u)^T A, kappa = <E(rho_u)^T C, E_v>
//   V (d2 rounds): E_hat sum E_v [alpha_s bw - 2^-d1 cu],
//                  bw = E(rho_w)^T B, cu = E(rho_u)^T C
// Everything between the transcript draws is stream-ordered device work; the
// host only runs the transcript (persistent.cu) and reads back kappa through
// an event while the next phase's kernel is already queued.
#include <chrono>
#include <cstdlib>
#include <vector>

#include "hostfield.h"
#include "phase.cuh"

namespace zkl {

template <class F>
static typename F::T half_p_plus_1() {  // (p + 1) / 2 in storage form
  typename F::T c;
  if constexpr (F::kId == 0) {
    uint64_t x[4] = {host::Fr::P[0], host::Fr::P[1], host::Fr::P[2], host::Fr::P[3]};
    // p + 1 (p odd: no carry past limb 0 except through 0xffff... limbs)
    unsigned __int128 cy = 1;
    for (int i = 0; i < 4; i++) {
      cy += x[i];
      x[i] = (uint64_t)cy;
      cy >>= 64;
    }
    for (int i = 0; i < 4; i++) x[i] = (x[i] >> 1) | (i < 3 ? x[i + 1] << 63 : 0);
    memcpy(&c, x, 32);
  } else {
    c = (M61::P + 1) / 2;
  }
  return host::For<F>::H::to_mont(c);
}

template <class F>
static Terms<F> prod2_terms(const typename F::T& coef) {
  Terms<F> tm;
  memset(&tm, 0, sizeof(tm));
  tm.nterms = 1;
  tm.degree = 3;
  tm.nf[0] = 2;
  tm.fi[0][0] = 0;
  tm.fi[0][1] = 1;
  tm.coef[0] = coef;
  return tm;
}

template <class F>
static void absorb_elem(HostTranscript& tr, const char* label, const typename F::T& v) {
  uint8_t b[32];
  host::to_canon<F>(b, v);
  tr.append_elem(label, b, F::kBytes);
}

template <class F>
int op_matmul_prove(int ta, const void* A, int tb, const void* B, int tc, const void* C, int d0,
                    int d1, int d2, uint8_t* state, uint8_t* rounds_out, uint8_t* point_out,
                    uint8_t* finals_out, cudaStream_t s) {
  using T = typename F::T;
  using H = typename host::For<F>::H;
  constexpr int nb = F::kBytes;
  if (d0 < 0 || d1 < 0 || d2 < 0 || d0 > 30 || d1 > 30 || d2 > 30 || d0 + d1 + d2 > 62) {
    set_error("matmul_prove: bad dims (%d,%d,%d)", d0, d1, d2);
    return kErrArg;
  }
  const uint64_t D0 = 1ull << d0, D1 = 1ull << d1, D2 = 1ull << d2;
  const int n = d0 + d1 + d2;
  // ZKL_TRACE: host timestamps at the phase boundaries (stderr)
  static const bool tracing = getenv("ZKL_TRACE") != nullptr;
  double tmark[8] = {0};
  auto mark = [&](int i) {
    if (tracing)
      tmark[i] = std::chrono::duration<double, std::micro>(
                     std::chrono::steady_clock::now().time_since_epoch())
                     .count();
  };
  mark(0);
  cudaEvent_t gev[8] = {};
  auto gmark = [&](int i) {
    if (tracing) {
      if (!gev[i]) cudaEventCreate(&gev[i]);
      cudaEventRecord(gev[i], s);
    }
  };
  gmark(0);
  HostTranscript tr;
  memcpy(tr.state, state, 64);

  // r_u, r_v (gadgets.py:241-242; transcript.py:44-45)
  std::vector<uint8_t> ru((size_t)d0 * nb), rv((size_t)d2 * nb);
  char label[64];
  for (int i = 0; i < d0; i++) {
    snprintf(label, sizeof(label), "matmul/r_u/%d", i);
    challenge_canon<F>(tr, label, ru.data() + (size_t)i * nb);
  }
  for (int i = 0; i < d2; i++) {
    snprintf(label, sizeof(label), "matmul/r_v/%d", i);
    challenge_canon<F>(tr, label, rv.data() + (size_t)i * nb);
  }
  // cneg = -2^-d1 (gadgets.py:246), claim absorbed (sumcheck.py:90-95)
  T inv = H::one();
  const T i2 = half_p_plus_1<F>();
  for (int i = 0; i < d1; i++) inv = H::mul(inv, i2);
  const T cneg = H::sub(H::zero(), inv);
  {
    const uint8_t zero = 0, one = 1;
    const uint8_t shape[3] = {3, (uint8_t)n, 2};
    const uint8_t f0[3] = {0, 1, 2}, f1[2] = {0, 3};
    tr.append_str("sumcheck/sum", &zero, 1);
    tr.append_str("sumcheck/shape", shape, 3);
    tr.append_str("sumcheck/coeff", &one, 1);
    tr.append_str("sumcheck/factors", f0, 3);
    absorb_elem<F>(tr, "sumcheck/coeff", cneg);
    tr.append_str("sumcheck/factors", f1, 2);
  }

  // device vectors
  const uint64_t sizes[] = {D2, D1, D0, D0, D0, D1, D2, D1, D2, 1, D0};
  enum { EV, BV, HV, EU, ERU, AV, CU, ERW, BW, KAP, CV, NBUF };
  uint64_t off[NBUF + 1];
  off[0] = 0;
  for (int i = 0; i < NBUF; i++) off[i + 1] = off[i] + ((sizes[i] + 3) & ~3ull);
  // every vector has its own slot (cv included: the side stream writes EU and
  // CV concurrently).  The side stream, its events and the side scratch arena
  // are per device, so matmul_prove is single-threaded per device: one host
  // thread proves on a device at a time (include/zkl_b200.h, threading).
  void* wsv;
  int rc = work_reserve(off[NBUF] * sizeof(T) + 64, &wsv, s);
  if (rc) return rc;
  T* base = (T*)wsv;
  auto buf = [&](int i) { return base + off[i]; };
  // profiler brackets (no-ops unless zkl_prof_enable)
  auto esz = [](int t) { return t == 1 ? 2.0 : t == 2 ? 4.0 : t == 3 ? 8.0 : (double)sizeof(T); };
  auto mv_on = [&](cudaStream_t st, int t, const void* M, uint64_t r_, uint64_t c_, int tr,
                   const T* xin, T* yout) {
    const int h = prof_open(kProfMatvec, (double)r_ * c_ * esz(t) + (double)(r_ + c_) * sizeof(T),
                            (double)r_ * c_, st);
    const int r2 = op_matvec<F>(t, M, r_, c_, tr, xin, yout, st);
    prof_close(h, st);
    return r2;
  };
  auto mv = [&](int t, const void* M, uint64_t r_, uint64_t c_, int tr, const T* xin, T* yout) {
    return mv_on(s, t, M, r_, c_, tr, xin, yout);
  };
  auto eq_on = [&](cudaStream_t st, T* dst, const T* p_, int m) {
    const int h = prof_open(kProfEq, (double)(1ull << m) * sizeof(T), (double)(1ull << m), st);
    const int r2 = op_eq_table<F>(dst, p_, m, st);
    prof_close(h, st);
    return r2;
  };
  auto eq = [&](T* dst, const T* p_, int m) { return eq_on(s, dst, p_, m); };
  // independent products of a phase's inputs run concurrently on the side
  // stream (its own scratch arena); fork / join through events
  const cudaStream_t side = side_stream();
  static thread_local cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (!ev_fork) {
    ZKL_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    ZKL_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  }
  auto fork = [&]() -> int {
    ZKL_CUDA(cudaEventRecord(ev_fork, s));
    ZKL_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
    return kOk;
  };
  auto join = [&]() -> int {
    ZKL_CUDA(cudaEventRecord(ev_join, side));
    ZKL_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
    return kOk;
  };
  std::vector<T> pt(64);
  auto load_point = [&](const uint8_t* canon, int m) {
    for (int i = 0; i < m; i++) pt[i] = host::from_canon<F>(canon + (size_t)i * nb);
    return pt.data();
  };

  // ---- U phase inputs: E_v, bv = B E_v, cv = C E_v, h = A bv - cv
  rc = eq(buf(EV), load_point(rv.data(), d2), d2);
  if (rc) return rc;
  gmark(1);
  // side: cv = C E_v and E_u; main: bv = B E_v, abv = A bv; then h = abv - cv
  if ((rc = fork())) return rc;
  if ((rc = mv_on(side, tc, C, D0, D2, 0, buf(EV), buf(CV)))) return rc;  // cv
  if ((rc = eq_on(side, buf(EU), load_point(ru.data(), d0), d0))) return rc;
  if ((rc = mv(tb, B, D1, D2, 0, buf(EV), buf(BV)))) return rc;
  if ((rc = mv(ta, A, D0, D1, 0, buf(BV), buf(HV)))) return rc;  // abv
  if ((rc = join())) return rc;
  if ((rc = op_axpy<F>(buf(HV), buf(HV), H::sub(H::zero(), H::one()), buf(CV), D0, s))) return rc;
  mark(1);
  gmark(2);
  uint8_t* rounds = rounds_out;
  uint8_t* point = point_out;
  // Phases are pipelined: run_phase returns once the last challenge is sent,
  // the next phase's inputs are enqueued behind the still-running kernel, and
  // the previous phase's finals (E_hat, alpha_s) are collected by the next
  // phase's prepare() when its first round is finished on the host.
  PhaseArgs<F> pu, pw, pv;
  void* tabs_u[2] = {buf(EU), buf(HV)};
  void* tabs_w[2] = {buf(AV), buf(BV)};
  void* tabs_v[3] = {buf(EV), buf(BW), buf(CU)};
  T e_hat = H::one(), alpha_s = H::one();
  bool have_e_hat = d0 == 0;
  auto get_e_hat = [&]() -> int {
    if (!have_e_hat) {
      T fin[2];
      int r = wait_phase_finals<F>(pu, fin, s);
      if (r) return r;
      e_hat = fin[0];
      have_e_hat = true;
    }
    return kOk;
  };
  if (d0) {
    pu.tables = tabs_u;
    pu.k = 2;
    pu.num_vars = d0;
    pu.tm = prod2_terms<F>(H::one());
    pu.post_mul = H::one();
    if ((rc = run_phase<F>(pu, tr, rounds, point, nullptr, s))) return rc;
  }
  mark(2);
  gmark(3);
  // ---- W phase inputs: E(rho_u), a = E^T A, cu = E^T C, kappa = <cu, E_v>
  if ((rc = eq(buf(ERU), load_point(point, d0), d0))) return rc;
  rounds += (size_t)d0 * 4 * nb;
  point += (size_t)d0 * nb;
  if ((rc = fork())) return rc;
  if ((rc = mv_on(side, tc, C, D0, D2, 1, buf(ERU), buf(CU)))) return rc;  // cu (side)
  if ((rc = mv(ta, A, D0, D1, 1, buf(ERU), buf(AV)))) return rc;
  if ((rc = join())) return rc;
  if ((rc = op_dot<F>(buf(KAP), buf(CU), buf(EV), D2, s))) return rc;
  static thread_local T* kap_host = nullptr;
  static thread_local cudaEvent_t kap_ev = nullptr;
  if (!kap_host) {
    ZKL_CUDA(cudaHostAlloc((void**)&kap_host, 64, cudaHostAllocDefault));
    ZKL_CUDA(cudaEventCreateWithFlags(&kap_ev, cudaEventDisableTiming));
  }
  ZKL_CUDA(cudaMemcpyAsync(kap_host, buf(KAP), sizeof(T), cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaEventRecord(kap_ev, s));
  mark(3);
  gmark(4);
  bool have_alpha = false;
  if (d1) {
    pw.tables = tabs_w;
    pw.k = 2;
    pw.num_vars = d1;
    pw.tm = prod2_terms<F>(H::one());
    pw.post_mul = H::one();
    pw.prepare = [&](std::vector<T>& adds) -> int {
      int r = get_e_hat();
      if (r) return r;
      pw.post_mul = e_hat;
      ZKL_CUDA(cudaEventSynchronize(kap_ev));
      const T kappa = *kap_host;
      adds.resize(d1);
      T c = H::mul(cneg, kappa);  // cneg 2^(d1-j-1) kappa, j = d1-1 .. 0
      for (int j = d1 - 1; j >= 0; j--) {
        adds[j] = c;
        c = H::add(c, c);
      }
      return kOk;
    };
    if ((rc = run_phase<F>(pw, tr, rounds, point, nullptr, s))) return rc;
  } else {
    uint8_t b[32];
    if ((rc = op_read<F>(b, buf(AV), 1, s))) return rc;
    alpha_s = host::from_canon<F>(b);
    have_alpha = true;
  }
  auto get_alpha = [&]() -> int {
    if (!have_alpha) {
      T fin[2];
      int r = wait_phase_finals<F>(pw, fin, s);
      if (r) return r;
      alpha_s = fin[0];
      have_alpha = true;
    }
    return kOk;
  };
  mark(4);
  gmark(5);
  // ---- V phase inputs: E(rho_w), bw = E^T B
  if ((rc = eq(buf(ERW), load_point(point, d1), d1))) return rc;
  rounds += (size_t)d1 * 4 * nb;
  point += (size_t)d1 * nb;
  if ((rc = mv(tb, B, D1, D2, 1, buf(ERW), buf(BW)))) return rc;
  mark(5);
  gmark(6);
  T fin_v[3];
  if (d2) {
    pv.tables = tabs_v;
    pv.k = 3;
    pv.num_vars = d2;
    Terms<F> tm;
    memset(&tm, 0, sizeof(tm));
    tm.nterms = 2;
    tm.degree = 3;
    tm.nf[0] = tm.nf[1] = 2;
    tm.fi[0][0] = 0;
    tm.fi[0][1] = 1;
    tm.fi[1][0] = 0;
    tm.fi[1][1] = 2;
    tm.coef[0] = H::one();  // alpha_s, set by prepare (host-applied coefficient)
    tm.coef[1] = cneg;
    pv.tm = tm;
    pv.post_mul = H::one();
    pv.prepare = [&](std::vector<T>&) -> int {
      int r = get_e_hat();
      if (r) return r;
      if ((r = get_alpha())) return r;
      pv.post_mul = e_hat;
      pv.tm.coef[0] = alpha_s;
      return kOk;
    };
    if ((rc = run_phase<F>(pv, tr, rounds, point, fin_v, s))) return rc;
  } else {
    if ((rc = get_e_hat()) || (rc = get_alpha())) return rc;
    uint8_t b[64];
    if ((rc = op_read<F>(b, buf(BW), 1, s))) return rc;
    if ((rc = op_read<F>(b + 32, buf(CU), 1, s))) return rc;
    fin_v[0] = H::one();
    fin_v[1] = host::from_canon<F>(b);
    fin_v[2] = host::from_canon<F>(b + 32);
  }
  const T finals[4] = {H::mul(e_hat, fin_v[0]), alpha_s, fin_v[1], fin_v[2]};
  for (int q = 0; q < 4; q++) host::to_canon<F>(finals_out + (size_t)q * nb, finals[q]);
  memcpy(state, tr.state, 64);
  mark(6);
  gmark(7);
  if (tracing) {
    cudaStreamSynchronize(s);
    float g[7];
    for (int i = 0; i < 7; i++) cudaEventElapsedTime(&g[i], gev[i], gev[i + 1]);
    fprintf(stderr,
            "[zkl trace] matmul (%d,%d,%d) GPU us: eq_v %.1f | mv(B,C,A)+axpy+eq_u %.1f | U %.1f | "
            "eq+mv(A^T,C^T)+dot %.1f | W %.1f | eq+mv(B^T) %.1f | V %.1f\n",
            d0, d1, d2, g[0] * 1e3, g[1] * 1e3, g[2] * 1e3, g[3] * 1e3, g[4] * 1e3, g[5] * 1e3,
            g[6] * 1e3);
    for (int i = 0; i < 8; i++) cudaEventDestroy(gev[i]);
  }
  if (tracing)
    fprintf(stderr,
            "[zkl trace] matmul (%d,%d,%d) us: draw+enqueue %.1f | U %.1f | enqueue W %.1f | "
            "W %.1f | enqueue V %.1f | V %.1f | total %.1f\n",
            d0, d1, d2, tmark[1] - tmark[0], tmark[2] - tmark[1], tmark[3] - tmark[2],
            tmark[4] - tmark[3], tmark[5] - tmark[4], tmark[6] - tmark[5], tmark[6] - tmark[0]);
  return kOk;
}

template int op_matmul_prove<Fr255>(int, const void*, int, const void*, int, const void*, int,
                                    int, int, uint8_t*, uint8_t*, uint8_t*, uint8_t*,
                                    cudaStream_t);
template int op_matmul_prove<M61>(int, const void*, int, const void*, int, const void*, int, int,
                                  int, uint8_t*, uint8_t*, uint8_t*, uint8_t*, cudaStream_t);

}  // namespace zkl
