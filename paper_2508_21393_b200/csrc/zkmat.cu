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
#include <functional>
#include <map>
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

// ---------------------------------------------------------------------------
// The phase-input sequences (eq tables, matvecs on two streams, small vector
// ops) are host-paced: a dozen launches and event calls per phase, each a
// few microseconds of host time, while the GPU work between them is shorter.
// They are replayed as CUDA graphs instead.  A sequence runs eagerly the first
// time it is seen for a set of operands and buffers (so every arena reaches
// its size), is captured the second time, and replayed after that; the eq
// points travel through pinned host slots copied to device memory by a node
// of the graph.  The profiler's event brackets and ZKL_TRACE need the eager
// path; ZKL_NO_GRAPHS=1 forces it.
struct GraphKey {
  int field, which, ta, tb, tc, d0, d1, d2, slot;
  const void *A, *B, *C, *base;
  cudaStream_t s;
  uint64_t gen;
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec = nullptr;
  int seen = 0;
  unsigned long long launches = 0;  // kernels inside (zkl_launch_count)
};
static std::vector<GraphEntry>& graph_cache() {
  static std::vector<GraphEntry> v;
  return v;
}
static bool graphs_allowed() {
  static const bool env_off = getenv("ZKL_NO_GRAPHS") != nullptr || getenv("ZKL_TRACE") != nullptr;
  return !env_off && !prof_on();
}
// a per-device stream to capture on (the caller's stream may be the legacy
// default stream, which cannot capture; the graph is launched on it)
static cudaStream_t capture_stream() {
  static std::map<int, cudaStream_t> m;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t& st = m[dev];
  if (!st) cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  return st;
}
// run body() through the cache entry for key: eagerly on s, or captured on
// the capture stream (set_stream(cs) points the body at it) and launched on s
template <class Body, class SetStream>
static int run_graphed(GraphKey key, cudaStream_t s, Body&& body, SetStream&& set_stream) {
  key.gen = arena_generation();
  auto& cache = graph_cache();
  GraphEntry* e = nullptr;
  for (auto& c : cache)
    if (!memcmp(&c.key, &key, sizeof(key))) e = &c;
  if (!e) {
    if (cache.size() >= 256) {  // bounded: drop the oldest half
      for (size_t i = 0; i < cache.size() / 2; i++)
        if (cache[i].exec) cudaGraphExecDestroy(cache[i].exec);
      cache.erase(cache.begin(), cache.begin() + cache.size() / 2);
    }
    cache.push_back(GraphEntry());
    e = &cache.back();
    e->key = key;
  }
  if (e->exec) {
    ZKL_CUDA(cudaGraphLaunch(e->exec, s));
    g_launches += e->launches;
    return kOk;
  }
  if (e->seen++ == 0) return body();  // eager: arenas and lazy state settle
  const unsigned long long l0 = g_launches;
  const cudaStream_t cs = capture_stream();
  ZKL_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
  set_stream(cs);
  const int rc = body();
  set_stream(s);
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
  if (rc || ce != cudaSuccess || arena_generation() != key.gen) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    if (rc) return rc;
    return body();  // capture failed or an arena moved: run it eagerly
  }
  cudaGraphExec_t exec = nullptr;
  ZKL_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  cudaGraphDestroy(graph);
  e->exec = exec;
  e->launches = g_launches - l0;
  g_launches = l0;
  ZKL_CUDA(cudaGraphLaunch(exec, s));
  g_launches += e->launches;
  return kOk;
}

// mapped pinned host slots for the eq points of the graphed sequences,
// [job parity][point] (a batch has two claims in flight): the eq kernel reads
// its point straight from host memory when it runs (one PCIe read per block,
// no copy-engine hop in front of it)
template <class F>
struct PointSlots {
  PointArg<F>* host = nullptr;
  PointArg<F>* dev = nullptr;  // the same memory, device view
  static constexpr int kN = 2 * 4;
  int ensure() {
    if (!host) {
      ZKL_CUDA(cudaHostAlloc((void**)&host, kN * sizeof(PointArg<F>), cudaHostAllocMapped));
      ZKL_CUDA(cudaHostGetDevicePointer((void**)&dev, host, 0));
    }
    return kOk;
  }
};

// flag = 1 if any of the n words is nonzero (benign racing stores of 1)
__global__ void k_any_nonzero(const uint64_t* v, uint64_t n, unsigned* flag) {
  bool nz = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    nz |= v[i] != 0;
  if (__any_sync(0xffffffffu, nz) && (threadIdx.x & 31) == 0) *flag = 1u;
}
static bool zero_phase_enabled() {
  static const bool on = getenv("ZKL_NO_ZERO_PHASE") == nullptr;
  return on;
}

// 32 bytes device -> mapped host memory by a kernel (kappa for the host)
__global__ void k_to_host32(uint4* dst, const uint4* src) {
  if (threadIdx.x < 2) dst[threadIdx.x] = src[threadIdx.x];
}
template <class F>
static PointSlots<F>& point_slots() {
  static thread_local PointSlots<F> p;
  return p;
}

// One claim's prover state.  begin() draws r_u / r_v, absorbs the claim and
// enqueues the U-phase inputs; prove() runs the U, W and V phases and returns
// once the last challenge is published (the V phase's finals still in
// flight); end() collects them.  A batch runs begin() of claim i+1 between
// prove() and end() of claim i, so the next claim's challenge draws and
// matvecs are queued behind the last fold of the previous one and the GPU
// never waits for the host between claims.  Device buffers are stream-ordered
// (claim i+1's writes queue behind claim i's kernels) and the pending finals
// arrive through the mailbox, not from device memory.
template <class F>
struct MatmulJob {
  using T = typename F::T;
  using H = typename host::For<F>::H;
  static constexpr int nb = F::kBytes;
  enum { EV, BV, HV, EU, ERU, AV, CU, ERW, BW, KAP, CV, NBUF };

  int ta = 0, tb = 0, tc = 0;
  const void *A = nullptr, *B = nullptr, *C = nullptr;
  int d0 = 0, d1 = 0, d2 = 0;
  uint8_t *rounds_out = nullptr, *point_out = nullptr, *finals_out = nullptr;
  cudaStream_t s = nullptr;
  HostTranscript* tr = nullptr;

  uint64_t D0 = 0, D1 = 0, D2 = 0;
  int n = 0;
  T cneg{};
  uint64_t off[NBUF + 1] = {};
  T* base = nullptr;
  std::vector<uint8_t> ru, rv;
  std::vector<T> pt = std::vector<T>(64);
  PhaseArgs<F> pu, pw, pv;
  T e_hat{}, alpha_s{}, fin_v[3] = {};
  bool have_e_hat = false, have_alpha = false;
  uint8_t *rounds = nullptr, *point = nullptr;
  int slot = 0;          // point-slot parity (a batch alternates it per claim)
  bool graphed = false;  // phase inputs through the CUDA-graph cache

  GraphKey key_for(int which) const {
    GraphKey k;
    memset(&k, 0, sizeof(k));
    k.field = F::kId;
    k.which = which; k.ta = ta; k.tb = tb; k.tc = tc; k.d0 = d0; k.d1 = d1; k.d2 = d2;
    k.slot = slot; k.A = A; k.B = B; k.C = C; k.base = base; k.s = s;
    return k;
  }
  // point p of this job's slot: host copy (filled now) and device copy (a
  // memcpy node refreshes it when the graph runs)
  PointArg<F>* host_pt(int p) { return point_slots<F>().host + slot * 4 + p; }
  PointArg<F>* dev_pt(int p) { return point_slots<F>().dev + slot * 4 + p; }
  void fill_point(int p, const uint8_t* canon, int m) {
    PointArg<F>* h = host_pt(p);
    for (int i = 0; i < m; i++) {
      h->r[i] = host::from_canon<F>(canon + (size_t)i * nb);
      h->omr[i] = H::sub(H::one(), h->r[i]);
    }
  }
  int eq_dev_on(cudaStream_t st, T* dst, int p, int m) {
    return op_eq_table_dev<F>(dst, dev_pt(p), m, slot * 4 + p, st);
  }

  // ZKL_TRACE: host and GPU timestamps at the phase boundaries (stderr)
  bool tracing = false;
  double tmark[8] = {0};
  cudaEvent_t gev[8] = {};

  static bool dims_ok(int a, int b, int c) {
    return a >= 0 && b >= 0 && c >= 0 && a <= 30 && b <= 30 && c <= 30 && a + b + c <= 62;
  }
  // device workspace: every vector has its own slot (cv included: the side
  // stream writes EU and CV concurrently).  The side stream, its events and
  // the side scratch arena are per device, so matmul proving is
  // single-threaded per device (include/zkl_b200.h, threading).
  static size_t work_bytes(int a, int b, int c) {
    const uint64_t sizes[NBUF] = {1ull << c, 1ull << b, 1ull << a, 1ull << a, 1ull << a,
                                  1ull << b, 1ull << c, 1ull << b, 1ull << c, 1, 1ull << a};
    uint64_t tot = 0;
    for (int i = 0; i < NBUF; i++) tot += (sizes[i] + 3) & ~3ull;
    return tot * sizeof(T) + 64;
  }
  T* buf(int i) { return base + off[i]; }
  void mark(int i) {
    if (tracing)
      tmark[i] = std::chrono::duration<double, std::micro>(
                     std::chrono::steady_clock::now().time_since_epoch())
                     .count();
  }
  void gmark(int i) {
    if (tracing) {
      if (!gev[i]) cudaEventCreate(&gev[i]);
      cudaEventRecord(gev[i], s);
    }
  }
  static double esz(int t) {
    return t == 1 ? 2.0 : t == 2 ? 4.0 : t == 3 ? 8.0 : (double)sizeof(T);
  }
  // profiler brackets (no-ops unless zkl_prof_enable)
  int mv_on(cudaStream_t st, int t, const void* M, uint64_t r_, uint64_t c_, int trn, const T* xin,
            T* yout) {
    const int h = prof_open(kProfMatvec, (double)r_ * c_ * esz(t) + (double)(r_ + c_) * sizeof(T),
                            (double)r_ * c_, st);
    const int r2 = op_matvec<F>(t, M, r_, c_, trn, xin, yout, st);
    prof_close(h, st);
    return r2;
  }
  int mv(int t, const void* M, uint64_t r_, uint64_t c_, int trn, const T* xin, T* yout) {
    return mv_on(s, t, M, r_, c_, trn, xin, yout);
  }
  int eq_on(cudaStream_t st, T* dst, const T* p_, int m) {
    const int h = prof_open(kProfEq, (double)(1ull << m) * sizeof(T), (double)(1ull << m), st);
    const int r2 = op_eq_table<F>(dst, p_, m, st);
    prof_close(h, st);
    return r2;
  }
  int eq(T* dst, const T* p_, int m) { return eq_on(s, dst, p_, m); }
  // independent products of a phase's inputs run concurrently on the side
  // stream (its own scratch arena); fork / join through events
  static cudaEvent_t& ev_fork() {
    static thread_local cudaEvent_t e = nullptr;
    return e;
  }
  static cudaEvent_t& ev_join() {
    static thread_local cudaEvent_t e = nullptr;
    return e;
  }
  int fork() {
    if (!ev_fork()) {
      ZKL_CUDA(cudaEventCreateWithFlags(&ev_fork(), cudaEventDisableTiming));
      ZKL_CUDA(cudaEventCreateWithFlags(&ev_join(), cudaEventDisableTiming));
    }
    ZKL_CUDA(cudaEventRecord(ev_fork(), s));
    ZKL_CUDA(cudaStreamWaitEvent(side_stream(), ev_fork(), 0));
    return kOk;
  }
  int join() {
    ZKL_CUDA(cudaEventRecord(ev_join(), side_stream()));
    ZKL_CUDA(cudaStreamWaitEvent(s, ev_join(), 0));
    return kOk;
  }
  const T* load_point(const uint8_t* canon, int m) {
    for (int i = 0; i < m; i++) pt[i] = host::from_canon<F>(canon + (size_t)i * nb);
    return pt.data();
  }
  int get_e_hat() {
    if (!have_e_hat) {
      T fin[2];
      int r = wait_phase_finals<F>(pu, fin, s);
      if (r) return r;
      e_hat = fin[0];
      have_e_hat = true;
    }
    return kOk;
  }
  int get_alpha() {
    if (!have_alpha) {
      T fin[2];
      int r = wait_phase_finals<F>(pw, fin, s);
      if (r) return r;
      alpha_s = fin[0];
      have_alpha = true;
    }
    return kOk;
  }
  // is the device vector v[0..n) all zero?  The check is queued now and
  // waited for (an event right behind it) only by check_zero_wait
  static unsigned*& zflag_host() {
    static thread_local unsigned* p = nullptr;
    return p;
  }
  static unsigned*& zflag_dev() {
    static thread_local unsigned* p = nullptr;
    return p;
  }
  static cudaEvent_t& zero_ev() {
    static thread_local cudaEvent_t e = nullptr;
    return e;
  }
  int check_zero_async(const T* v, uint64_t n) {
    if (!zflag_host()) {
      ZKL_CUDA(cudaHostAlloc((void**)&zflag_host(), 64, cudaHostAllocMapped));
      ZKL_CUDA(cudaHostGetDevicePointer((void**)&zflag_dev(), zflag_host(), 0));
      ZKL_CUDA(cudaEventCreateWithFlags(&zero_ev(), cudaEventDisableTiming));
    }
    *reinterpret_cast<volatile unsigned*>(zflag_host()) = 0;
    const uint64_t words = n * sizeof(T) / 8;
    unsigned blocks = (unsigned)((words + 255) / 256);
    if (blocks > 2 * kSMs) blocks = 2 * kSMs;
    k_any_nonzero<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint64_t*>(v), words,
                                         zflag_dev());
    ZKL_LAUNCH_CHECK();
    ZKL_CUDA(cudaEventRecord(zero_ev(), s));
    return kOk;
  }
  int check_zero_wait(bool* zero) {
    ZKL_CUDA(cudaEventSynchronize(zero_ev()));
    *zero = *reinterpret_cast<volatile unsigned*>(zflag_host()) == 0;
    return kOk;
  }
  static T*& kap_host() {
    static thread_local T* p = nullptr;
    return p;
  }
  static T*& kap_dev() {
    static thread_local T* p = nullptr;
    return p;
  }
  static cudaEvent_t& kap_ev() {
    static thread_local cudaEvent_t e = nullptr;
    return e;
  }

  int begin() {
    if (!dims_ok(d0, d1, d2)) {
      set_error("matmul_prove: bad dims (%d,%d,%d)", d0, d1, d2);
      return kErrArg;
    }
    D0 = 1ull << d0;
    D1 = 1ull << d1;
    D2 = 1ull << d2;
    n = d0 + d1 + d2;
    tracing = getenv("ZKL_TRACE") != nullptr;
    mark(0);
    gmark(0);
    // r_u, r_v (gadgets.py:241-242; transcript.py:44-45)
    ru.resize((size_t)d0 * nb);
    rv.resize((size_t)d2 * nb);
    char label[64];
    for (int i = 0; i < d0; i++) {
      snprintf(label, sizeof(label), "matmul/r_u/%d", i);
      challenge_canon<F>(*tr, label, ru.data() + (size_t)i * nb);
    }
    for (int i = 0; i < d2; i++) {
      snprintf(label, sizeof(label), "matmul/r_v/%d", i);
      challenge_canon<F>(*tr, label, rv.data() + (size_t)i * nb);
    }
    // cneg = -2^-d1 (gadgets.py:246), claim absorbed (sumcheck.py:90-95)
    T inv = H::one();
    const T i2 = half_p_plus_1<F>();
    for (int i = 0; i < d1; i++) inv = H::mul(inv, i2);
    cneg = H::sub(H::zero(), inv);
    {
      const uint8_t zero = 0, one = 1;
      const uint8_t shape[3] = {3, (uint8_t)n, 2};
      const uint8_t f0[3] = {0, 1, 2}, f1[2] = {0, 3};
      tr->append_str("sumcheck/sum", &zero, 1);
      tr->append_str("sumcheck/shape", shape, 3);
      tr->append_str("sumcheck/coeff", &one, 1);
      tr->append_str("sumcheck/factors", f0, 3);
      absorb_elem<F>(*tr, "sumcheck/coeff", cneg);
      tr->append_str("sumcheck/factors", f1, 2);
    }
    const uint64_t sizes[NBUF] = {D2, D1, D0, D0, D0, D1, D2, D1, D2, 1, D0};
    off[0] = 0;
    for (int i = 0; i < NBUF; i++) off[i + 1] = off[i] + ((sizes[i] + 3) & ~3ull);
    void* wsv;
    int rc = work_reserve(work_bytes(d0, d1, d2), &wsv, s);
    if (rc) return rc;
    base = (T*)wsv;
    // ---- U phase inputs: E_v, bv = B E_v, cv = C E_v, h = A bv - cv
    graphed = graphs_allowed() && d0 >= 1 && d0 <= 16 && d1 >= 1 && d1 <= 16 && d2 >= 1 &&
              d2 <= 16 && point_slots<F>().ensure() == kOk;
    auto u_inputs = [&]() -> int {
      int r;
      if (graphed) {
        if ((r = eq_dev_on(s, buf(EV), 0, d2))) return r;
      } else if ((r = eq(buf(EV), load_point(rv.data(), d2), d2))) {
        return r;
      }
      gmark(1);
      // side: cv = C E_v and E_u; main: bv = B E_v, abv = A bv; then h = abv - cv
      if ((r = fork())) return r;
      if (graphed) {
        if ((r = eq_dev_on(side_stream(), buf(EU), 1, d0))) return r;
      } else if ((r = eq_on(side_stream(), buf(EU), load_point(ru.data(), d0), d0))) {
        return r;
      }
      if ((r = mv_on(side_stream(), tc, C, D0, D2, 0, buf(EV), buf(CV)))) return r;  // cv
      if ((r = mv(tb, B, D1, D2, 0, buf(EV), buf(BV)))) return r;
      if ((r = mv(ta, A, D0, D1, 0, buf(BV), buf(HV)))) return r;  // abv
      if ((r = join())) return r;
      return op_axpy<F>(buf(HV), buf(HV), H::sub(H::zero(), H::one()), buf(CV), D0, s);
    };
    if (graphed) {
      fill_point(0, rv.data(), d2);
      fill_point(1, ru.data(), d0);
      if ((rc = run_graphed(key_for(0), s, u_inputs, [this](cudaStream_t st) { s = st; }))) return rc;
    } else if ((rc = u_inputs())) {
      return rc;
    }
    mark(1);
    gmark(2);
    return kOk;
  }

  // Phases are pipelined: run_phase returns once the last challenge is sent,
  // the next phase's inputs are enqueued behind the still-running kernel, and
  // the previous phase's finals (E_hat, alpha_s) are collected by the next
  // phase's prepare() when its first round is finished on the host.
  int prove() {
    int rc;
    rounds = rounds_out;
    point = point_out;
    e_hat = H::one();
    alpha_s = H::one();
    have_e_hat = d0 == 0;
    have_alpha = false;
    void* tabs_u[2] = {buf(EU), buf(HV)};
    void* tabs_w[2] = {buf(AV), buf(BV)};
    void* tabs_v[3] = {buf(EV), buf(BW), buf(CU)};
    if (!kap_host()) {
      ZKL_CUDA(cudaHostAlloc((void**)&kap_host(), 64, cudaHostAllocMapped));
      ZKL_CUDA(cudaHostGetDevicePointer((void**)&kap_dev(), kap_host(), 0));
      ZKL_CUDA(cudaEventCreateWithFlags(&kap_ev(), cudaEventDisableTiming));
    }
    // ---- W phase inputs: E(rho_u), a = E^T A, cu = E^T C, kappa = <cu, E_v>
    auto launch_w = [&](const uint8_t* rho_u) -> int {
      auto w_inputs = [&]() -> int {
        int r;
        if (graphed) {
          if ((r = eq_dev_on(s, buf(ERU), 2, d0))) return r;
        } else if ((r = eq(buf(ERU), load_point(rho_u, d0), d0))) {
          return r;
        }
        if ((r = fork())) return r;
        if ((r = mv_on(side_stream(), tc, C, D0, D2, 1, buf(ERU), buf(CU)))) return r;  // cu
        if ((r = mv(ta, A, D0, D1, 1, buf(ERU), buf(AV)))) return r;
        if ((r = join())) return r;
        if ((r = op_dot<F>(buf(KAP), buf(CU), buf(EV), D2, s))) return r;
        k_to_host32<<<1, 32, 0, s>>>(reinterpret_cast<uint4*>(kap_dev()),
                                     reinterpret_cast<const uint4*>(buf(KAP)));
        ZKL_LAUNCH_CHECK();
        return kOk;
      };
      int r;
      if (graphed) {
        fill_point(2, rho_u, d0);
        if ((r = run_graphed(key_for(1), s, w_inputs, [this](cudaStream_t st) { s = st; })))
          return r;
      } else if ((r = w_inputs())) {
        return r;
      }
      ZKL_CUDA(cudaEventRecord(kap_ev(), s));
      return kOk;
    };
    bool w_launched = false;
    if (d0) {
      bool zero = false;
      if (zero_phase_enabled()) {
        // A true claim (C = A B) has h = A (B E_v) - C E_v = 0 identically, so
        // every U-phase round polynomial E_u h is the zero polynomial: the
        // rounds are the transcript's alone (4 zero evaluations, then the
        // challenge), and the folded finals are E_u(rho) = eq(r_u, rho) and
        // h(rho) = 0.  Same bytes as the device rounds.  The host rounds run
        // speculatively while the device still computes h, and the W inputs
        // for the resulting rho_u are queued right behind the zero check; a
        // false claim (h != 0) restores the transcript, runs the device
        // rounds and recomputes the W inputs
        // (tests/test_gpu_parity.py::test_matmul_factored_vs_oracle).
        uint8_t saved[64];
        memcpy(saved, tr->state, 64);
        memset(rounds, 0, (size_t)d0 * 4 * nb);
        const uint8_t zb = 0;
        T eq = H::one();
        for (int j = 0; j < d0; j++) {
          for (int x = 0; x < 4; x++) tr->append_elem("sumcheck/eval", &zb, 1);
          challenge_canon<F>(*tr, "sumcheck/round", point + (size_t)j * nb);
          const T r = host::from_canon<F>(ru.data() + (size_t)j * nb);
          const T rho = host::from_canon<F>(point + (size_t)j * nb);
          // eq(r, rho) = r rho + (1 - r)(1 - rho)
          const T t = H::add(H::mul(r, rho), H::mul(H::sub(H::one(), r), H::sub(H::one(), rho)));
          eq = H::mul(eq, t);
        }
        if ((rc = check_zero_async(buf(HV), D0))) return rc;
        if ((rc = launch_w(point))) return rc;
        w_launched = true;
        if ((rc = check_zero_wait(&zero))) return rc;
        if (zero) {
          e_hat = eq;
          have_e_hat = true;
        } else {
          memcpy(tr->state, saved, 64);
          w_launched = false;
        }
      }
      if (!zero) {
        pu.tables = tabs_u;
        pu.k = 2;
        pu.num_vars = d0;
        pu.tm = prod2_terms<F>(H::one());
        pu.post_mul = H::one();
        pu.host_tail = host_tail_default();
        if ((rc = run_phase<F>(pu, *tr, rounds, point, nullptr, s))) return rc;
      }
    }
    mark(2);
    gmark(3);
    if (!w_launched && (rc = launch_w(point))) return rc;
    rounds += (size_t)d0 * 4 * nb;
    point += (size_t)d0 * nb;
    mark(3);
    gmark(4);
    if (d1) {
      pw.tables = tabs_w;
      pw.k = 2;
      pw.num_vars = d1;
      pw.tm = prod2_terms<F>(H::one());
      pw.post_mul = H::one();
      pw.host_tail = host_tail_default();
      pw.prepare = [this](std::vector<T>& adds) -> int {
        int r = get_e_hat();
        if (r) return r;
        pw.post_mul = e_hat;
        ZKL_CUDA(cudaEventSynchronize(kap_ev()));
        const T kappa = *kap_host();
        adds.resize(d1);
        T c = H::mul(cneg, kappa);  // cneg 2^(d1-j-1) kappa, j = d1-1 .. 0
        for (int j = d1 - 1; j >= 0; j--) {
          adds[j] = c;
          c = H::add(c, c);
        }
        return kOk;
      };
      if ((rc = run_phase<F>(pw, *tr, rounds, point, nullptr, s))) return rc;
    } else {
      uint8_t b[32];
      if ((rc = op_read<F>(b, buf(AV), 1, s))) return rc;
      alpha_s = host::from_canon<F>(b);
      have_alpha = true;
    }
    mark(4);
    gmark(5);
    // ---- V phase inputs: E(rho_w), bw = E^T B
    const uint8_t* rho_w = point;
    auto v_inputs = [&]() -> int {
      int r;
      if (graphed) {
        if ((r = eq_dev_on(s, buf(ERW), 3, d1))) return r;
      } else if ((r = eq(buf(ERW), load_point(rho_w, d1), d1))) {
        return r;
      }
      return mv(tb, B, D1, D2, 1, buf(ERW), buf(BW));
    };
    if (graphed) {
      fill_point(3, rho_w, d1);
      if ((rc = run_graphed(key_for(2), s, v_inputs, [this](cudaStream_t st) { s = st; }))) return rc;
    } else if ((rc = v_inputs())) {
      return rc;
    }
    rounds += (size_t)d1 * 4 * nb;
    point += (size_t)d1 * nb;
    mark(5);
    gmark(6);
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
      pv.host_tail = host_tail_default();
      pv.prepare = [this](std::vector<T>&) -> int {
        int r = get_e_hat();
        if (r) return r;
        if ((r = get_alpha())) return r;
        pv.post_mul = e_hat;
        pv.tm.coef[0] = alpha_s;
        return kOk;
      };
      // the V finals are collected by end()
      if ((rc = run_phase<F>(pv, *tr, rounds, point, nullptr, s))) return rc;
    } else {
      if ((rc = get_e_hat()) || (rc = get_alpha())) return rc;
      uint8_t b[64];
      if ((rc = op_read<F>(b, buf(BW), 1, s))) return rc;
      if ((rc = op_read<F>(b + 32, buf(CU), 1, s))) return rc;
      fin_v[0] = H::one();
      fin_v[1] = host::from_canon<F>(b);
      fin_v[2] = host::from_canon<F>(b + 32);
    }
    return kOk;
  }

  int end() {
    int rc;
    if (d2 && (rc = wait_phase_finals<F>(pv, fin_v, s))) return rc;
    const T finals[4] = {H::mul(e_hat, fin_v[0]), alpha_s, fin_v[1], fin_v[2]};
    for (int q = 0; q < 4; q++) host::to_canon<F>(finals_out + (size_t)q * nb, finals[q]);
    mark(6);
    gmark(7);
    if (tracing) report();
    return kOk;
  }

  void report() {
    cudaStreamSynchronize(s);
    float g[7];
    for (int i = 0; i < 7; i++) cudaEventElapsedTime(&g[i], gev[i], gev[i + 1]);
    fprintf(stderr,
            "[zkl trace] matmul (%d,%d,%d) GPU us: eq_v %.1f | mv(B,C,A)+axpy+eq_u %.1f | U %.1f | "
            "eq+mv(A^T,C^T)+dot %.1f | W %.1f | eq+mv(B^T) %.1f | V %.1f\n",
            d0, d1, d2, g[0] * 1e3, g[1] * 1e3, g[2] * 1e3, g[3] * 1e3, g[4] * 1e3, g[5] * 1e3,
            g[6] * 1e3);
    for (int i = 0; i < 8; i++) cudaEventDestroy(gev[i]);
    fprintf(stderr,
            "[zkl trace] matmul (%d,%d,%d) us: draw+enqueue %.1f | U %.1f | enqueue W %.1f | "
            "W %.1f | enqueue V %.1f | V %.1f | total %.1f\n",
            d0, d1, d2, tmark[1] - tmark[0], tmark[2] - tmark[1], tmark[3] - tmark[2],
            tmark[4] - tmark[3], tmark[5] - tmark[4], tmark[6] - tmark[5], tmark[6] - tmark[0]);
  }
};

template <class F>
int op_matmul_prove(int ta, const void* A, int tb, const void* B, int tc, const void* C, int d0,
                    int d1, int d2, uint8_t* state, uint8_t* rounds_out, uint8_t* point_out,
                    uint8_t* finals_out, cudaStream_t s) {
  HostTranscript tr;
  memcpy(tr.state, state, 64);
  MatmulJob<F> job;
  job.ta = ta; job.tb = tb; job.tc = tc;
  job.A = A; job.B = B; job.C = C;
  job.d0 = d0; job.d1 = d1; job.d2 = d2;
  job.rounds_out = rounds_out; job.point_out = point_out; job.finals_out = finals_out;
  job.s = s;
  job.tr = &tr;
  int rc;
  if ((rc = job.begin()) || (rc = job.prove()) || (rc = job.end())) return rc;
  memcpy(state, tr.state, 64);
  return kOk;
}

// Transcript records appended before a claim: u16le |label| || label ||
// u64le |data| || data, repeated (the framing of transcript.py:13-35).
static int append_records(HostTranscript& tr, const uint8_t* p, uint64_t len) {
  uint64_t o = 0;
  while (o < len) {
    if (len - o < 2) return kErrArg;
    const size_t ll = (size_t)p[o] | ((size_t)p[o + 1] << 8);
    o += 2;
    if (len - o < ll + 8) return kErrArg;
    const char* label = (const char*)(p + o);
    o += ll;
    uint64_t dl = 0;
    for (int i = 0; i < 8; i++) dl |= (uint64_t)p[o + i] << (8 * i);
    o += 8;
    if (len - o < dl) return kErrArg;
    tr.append(label, ll, p + o, (size_t)dl);
    o += dl;
  }
  return kOk;
}

template <class F>
int op_matmul_prove_batch(int nclaims, const int* types, const void* const* mats, const int* dims,
                          const uint8_t* pre, const uint64_t* pre_off, uint8_t* state,
                          uint8_t* rounds_out, uint8_t* point_out, uint8_t* finals_out,
                          cudaStream_t s) {
  constexpr int nb = F::kBytes;
  if (nclaims < 0) return kErrArg;
  if (nclaims == 0) return kOk;
  HostTranscript tr;
  memcpy(tr.state, state, 64);
  // the largest claim's workspace up front: growing it mid-batch would
  // synchronise the stream
  size_t want = 0;
  for (int i = 0; i < nclaims; i++) {
    const int* d = dims + 3 * i;
    if (!MatmulJob<F>::dims_ok(d[0], d[1], d[2])) {
      set_error("matmul_prove_batch: claim %d has bad dims (%d,%d,%d)", i, d[0], d[1], d[2]);
      return kErrArg;
    }
    const size_t w = MatmulJob<F>::work_bytes(d[0], d[1], d[2]);
    want = w > want ? w : want;
  }
  void* ws;
  int rc = work_reserve(want, &ws, s);
  if (rc) return rc;
  std::vector<MatmulJob<F>> jobs(2);
  size_t roff = 0, poff = 0;
  auto setup = [&](MatmulJob<F>& j, int i) -> int {
    j = MatmulJob<F>();
    const int* d = dims + 3 * i;
    j.ta = types[3 * i]; j.tb = types[3 * i + 1]; j.tc = types[3 * i + 2];
    j.A = mats[3 * i]; j.B = mats[3 * i + 1]; j.C = mats[3 * i + 2];
    j.d0 = d[0]; j.d1 = d[1]; j.d2 = d[2];
    j.rounds_out = rounds_out + roff * 4 * nb;
    j.point_out = point_out + poff * nb;
    j.finals_out = finals_out + (size_t)i * 4 * nb;
    roff += (size_t)(d[0] + d[1] + d[2]);
    poff += (size_t)(d[0] + d[1] + d[2]);
    j.s = s;
    j.tr = &tr;
    j.slot = i & 1;
    if (pre && pre_off) {
      const int r = append_records(tr, pre + pre_off[i], pre_off[i + 1] - pre_off[i]);
      if (r) {
        set_error("matmul_prove_batch: malformed transcript records before claim %d", i);
        return r;
      }
    }
    return j.begin();
  };
  if ((rc = setup(jobs[0], 0))) return rc;
  for (int i = 0; i < nclaims; i++) {
    MatmulJob<F>& cur = jobs[i & 1];
    if ((rc = cur.prove())) return rc;
    // the next claim's draws and inputs queue behind this claim's last fold
    if (i + 1 < nclaims && (rc = setup(jobs[(i + 1) & 1], i + 1))) return rc;
    if ((rc = cur.end())) return rc;
  }
  memcpy(state, tr.state, 64);
  return kOk;
}

template int op_matmul_prove<Fr255>(int, const void*, int, const void*, int, const void*, int,
                                    int, int, uint8_t*, uint8_t*, uint8_t*, uint8_t*,
                                    cudaStream_t);
template int op_matmul_prove<M61>(int, const void*, int, const void*, int, const void*, int, int,
                                  int, uint8_t*, uint8_t*, uint8_t*, uint8_t*, cudaStream_t);
template int op_matmul_prove_batch<Fr255>(int, const int*, const void* const*, const int*,
                                          const uint8_t*, const uint64_t*, uint8_t*, uint8_t*,
                                          uint8_t*, uint8_t*, cudaStream_t);
template int op_matmul_prove_batch<M61>(int, const int*, const void* const*, const int*,
                                        const uint8_t*, const uint64_t*, uint8_t*, uint8_t*,
                                        uint8_t*, uint8_t*, cudaStream_t);

}  // namespace zkl
