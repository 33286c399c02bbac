// Element-wise field kernels: Montgomery conversion, int -> field lift,
// eq-table, fold, axpy, dot; plus the scratch arena and error plumbing.
//
// Reference: mle.py:50-82 (fold_table, eq_table), field.py:49-55 (signed
// lift), quantize.py:176-183 (row-major zero-padded residues).
#include <stdarg.h>
#include <string.h>

#include <map>
#include <vector>
#include <mutex>

#include "ops.cuh"

namespace zkl {

// ---------------------------------------------------------------------------
// error + scratch
unsigned long long g_launches = 0;
static thread_local char g_err[512];
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* get_error() { return g_err; }

// bumped whenever a scratch or work arena moves: device pointers captured in a
// CUDA graph (zkmat.cu) are valid only for the generation they were taken in
static uint64_t g_arena_gen = 0;
static std::map<int, Scratch>& arenas() {
  static std::map<int, Scratch> m;
  return m;
}
Scratch& scratch_for_current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return arenas()[dev];
}
// A per-device side stream for independent work inside one call (the zkMat
// driver's concurrent matrix-vector products); work on it takes its own
// scratch arena, so it never aliases the main stream's.
static std::map<int, cudaStream_t>& side_streams() {
  static std::map<int, cudaStream_t> m;
  return m;
}
static std::map<int, Scratch>& side_arenas() {
  static std::map<int, Scratch> m;
  return m;
}
cudaStream_t side_stream() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t& st = side_streams()[dev];
  if (!st) cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  return st;
}
int scratch_reserve(size_t bytes, void** out, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = side_streams().find(dev);
  const bool side = s != nullptr && it != side_streams().end() && it->second == s;
  Scratch& a = side ? side_arenas()[dev] : scratch_for_current_device();
  if (bytes > a.bytes) {
    if (a.ptr) {
      ZKL_CUDA(cudaStreamSynchronize(s));
      ZKL_CUDA(cudaFree(a.ptr));
      a.ptr = nullptr;
      a.bytes = 0;
    }
    size_t want = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 4;
    ZKL_CUDA(cudaMalloc(&a.ptr, want));
    a.bytes = want;
    ++g_arena_gen;
  }
  *out = a.ptr;
  return kOk;
}
uint64_t arena_generation() { return g_arena_gen; }
// ---------------------------------------------------------------------------
// CUDA-event profiler
struct ProfRec {
  cudaEvent_t a = nullptr, b = nullptr;
  int kind = 0;
  double bytes = 0, units = 0;
};
static std::vector<ProfRec>& prof_recs() {
  static std::vector<ProfRec> v;
  return v;
}
static bool g_prof = false;
static std::vector<cudaEvent_t>& event_pool() {  // recycled: no create/destroy per launch
  static std::vector<cudaEvent_t> v;
  return v;
}
static cudaEvent_t pool_get() {
  auto& p = event_pool();
  if (p.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = p.back();
  p.pop_back();
  return e;
}
bool prof_on() { return g_prof; }
int prof_open(int kind, double bytes, double units, cudaStream_t s) {
  if (!g_prof) return -1;
  ProfRec r;
  r.kind = kind;
  r.bytes = bytes;
  r.units = units;
  r.a = pool_get();
  r.b = pool_get();
  cudaEventRecord(r.a, s);
  prof_recs().push_back(r);
  return (int)prof_recs().size() - 1;
}
void prof_close(int h, cudaStream_t s) {
  if (h < 0 || h >= (int)prof_recs().size()) return;
  cudaEventRecord(prof_recs()[h].b, s);
}
void prof_enable(bool on) { g_prof = on; }
// sums over the records of `kind` (syncs on their events); clears them
void prof_collect(int kind, double* ms, double* bytes, double* units, uint64_t* count) {
  double t = 0, by = 0, un = 0;
  uint64_t n = 0;
  auto& v = prof_recs();
  std::vector<ProfRec> keep;
  for (auto& r : v) {
    if (r.kind != kind) {
      keep.push_back(r);
      continue;
    }
    float e = 0;
    cudaEventSynchronize(r.b);
    if (cudaEventElapsedTime(&e, r.a, r.b) != cudaSuccess) {
      e = 0;  // bracket never closed: do not leave a sticky error behind
      cudaGetLastError();
    }
    t += e;
    by += r.bytes;
    un += r.units;
    n++;
    event_pool().push_back(r.a);
    event_pool().push_back(r.b);
  }
  v.swap(keep);
  *ms = t;
  *bytes = by;
  *units = un;
  *count = n;
}

int work_reserve(size_t bytes, void** out, cudaStream_t s) {
  Scratch& a = scratch_for_current_device();
  if (bytes > a.work_bytes) {
    if (a.work) {
      ZKL_CUDA(cudaStreamSynchronize(s));
      ZKL_CUDA(cudaFree(a.work));
      a.work = nullptr;
      a.work_bytes = 0;
    }
    size_t want = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 4;
    ZKL_CUDA(cudaMalloc(&a.work, want));
    a.work_bytes = want;
    ++g_arena_gen;
  }
  *out = a.work;
  return kOk;
}
int fixed_words(void** out) {
  Scratch& a = scratch_for_current_device();
  if (!a.fixed) {
    ZKL_CUDA(cudaMalloc(&a.fixed, 4096));
    ZKL_CUDA(cudaMemset(a.fixed, 0, 4096));
  }
  *out = a.fixed;
  return kOk;
}
static std::map<int, std::pair<Mailbox*, Mailbox*>>& mailboxes() {
  static std::map<int, std::pair<Mailbox*, Mailbox*>> m;
  return m;
}
int mailbox_for_current_device(Mailbox** host, Mailbox** dev) {
  int d = 0;
  cudaGetDevice(&d);
  auto& e = mailboxes()[d];
  if (!e.first) {
    void* h = nullptr;
    ZKL_CUDA(cudaHostAlloc(&h, sizeof(Mailbox), cudaHostAllocMapped | cudaHostAllocPortable));
    memset(h, 0, sizeof(Mailbox));
    void* dp = nullptr;
    ZKL_CUDA(cudaHostGetDevicePointer(&dp, h, 0));
    e.first = (Mailbox*)h;
    e.second = (Mailbox*)dp;
  }
  *host = e.first;
  *dev = e.second;
  return kOk;
}
int pinned_reserve(size_t bytes, void** out) {
  Scratch& a = scratch_for_current_device();
  if (bytes > a.pinned_bytes) {
    if (a.pinned) ZKL_CUDA(cudaFreeHost(a.pinned));
    size_t want = bytes < 65536 ? 65536 : bytes;
    ZKL_CUDA(cudaHostAlloc(&a.pinned, want, cudaHostAllocDefault));
    a.pinned_bytes = want;
  }
  *out = a.pinned;
  return kOk;
}

// ---------------------------------------------------------------------------
template <class F>
__global__ void k_to_mont(typename F::T* dst, const typename F::T* src, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    typename F::T v = src[i];
    // canonical inputs are < p; reduce once defensively for Fr255 inputs < 2^256
    dst[i] = F::to_mont(v);
  }
}
template <class F>
__global__ void k_from_mont(typename F::T* dst, const typename F::T* src, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = F::from_mont(src[i]);
}
template <class F, class I>
__global__ void k_lift(typename F::T* dst, const I* src, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = F::from_i64((int64_t)src[i]);
}

// pair-table compression (gadgets.py:659-666, tables.py:131-140):
// dst[i] = x[i] + alpha * y[i] with signed integer columns lifted on the fly
template <class F, class IX, class IY>
__global__ void k_pair_combine(typename F::T* dst, const IX* x, const IY* y, uint64_t n,
                               typename F::T alpha) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = F::add(F::from_i64((int64_t)x[i]), F::mul(alpha, F::from_i64((int64_t)y[i])));
}

template <class F, class IX>
static int pair_combine_y(typename F::T* d, const IX* x, const void* y, int ty, uint64_t n,
                          typename F::T a, cudaStream_t s) {
  const unsigned g = grid_for(n, 256);
  switch (ty) {
    case 1: k_pair_combine<F, IX, int16_t><<<g, 256, 0, s>>>(d, x, (const int16_t*)y, n, a); break;
    case 2: k_pair_combine<F, IX, int32_t><<<g, 256, 0, s>>>(d, x, (const int32_t*)y, n, a); break;
    case 3: k_pair_combine<F, IX, int64_t><<<g, 256, 0, s>>>(d, x, (const int64_t*)y, n, a); break;
    default: set_error("pair_combine: bad y type %d", ty); return kErrArg;
  }
  ZKL_LAUNCH_CHECK();
  return kOk;
}

// int16 x int16 columns: two 2^16-entry lookup tables (lift(v) and
// alpha * lift(v) for every int16 v, 2 MB each, L2-resident), so each secret
// entry costs two L2 loads and one field add instead of three Montgomery
// products.
template <class F>
__global__ void k_pair_luts(typename F::T* lx, typename F::T* ly, typename F::T alpha) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 65536) {
    const typename F::T v = F::from_i64((int64_t)i - 32768);
    lx[i] = v;
    ly[i] = F::mul(alpha, v);
  }
}
template <class F>
__global__ void k_pair_combine_lut(typename F::T* dst, const int16_t* x, const int16_t* y,
                                   uint64_t n, const typename F::T* lx, const typename F::T* ly) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = F::add(lx[(int)x[i] + 32768], ly[(int)y[i] + 32768]);
}

template <class F>
int op_pair_combine(void* dst, const void* x, int tx, const void* y, int ty, uint64_t n,
                    typename F::T alpha, cudaStream_t s) {
  if (!n) return kOk;
  using T = typename F::T;
  T* d = (T*)dst;
  if (tx == 1 && ty == 1 && n >= (1u << 18)) {
    void* ws;
    int rc = scratch_reserve(2 * 65536 * sizeof(T), &ws, s);
    if (rc) return rc;
    T* lx = (T*)ws;
    T* ly = lx + 65536;
    k_pair_luts<F><<<256, 256, 0, s>>>(lx, ly, alpha);
    ZKL_LAUNCH_CHECK();
    k_pair_combine_lut<F><<<grid_for(n, 256), 256, 0, s>>>(d, (const int16_t*)x,
                                                           (const int16_t*)y, n, lx, ly);
    ZKL_LAUNCH_CHECK();
    return kOk;
  }
  switch (tx) {
    case 1: return pair_combine_y<F, int16_t>(d, (const int16_t*)x, y, ty, n, alpha, s);
    case 2: return pair_combine_y<F, int32_t>(d, (const int32_t*)x, y, ty, n, alpha, s);
    case 3: return pair_combine_y<F, int64_t>(d, (const int64_t*)x, y, ty, n, alpha, s);
  }
  set_error("pair_combine: bad x type %d", tx);
  return kErrArg;
}

template <class F>
int op_to_mont(void* dst, const void* src, uint64_t n, cudaStream_t s) {
  if (!n) return kOk;
  k_to_mont<F><<<grid_for(n, 256), 256, 0, s>>>((typename F::T*)dst,
                                                 (const typename F::T*)src, n);
  ZKL_LAUNCH_CHECK();
  return kOk;
}
template <class F>
int op_from_mont(void* dst, const void* src, uint64_t n, cudaStream_t s) {
  if (!n) return kOk;
  k_from_mont<F><<<grid_for(n, 256), 256, 0, s>>>((typename F::T*)dst,
                                                   (const typename F::T*)src, n);
  ZKL_LAUNCH_CHECK();
  return kOk;
}
// Fr255 lift through look-up tables (one Montgomery product per table entry,
// built once per process and device, 10 MB, L2-resident): int16 values index
// a signed 2^16-entry table; wider values are split into 16-bit chunks c_k of
// |x| and summed as sum_k T_k[c_k] with T_k[c] = (c 2^(16k)) R mod p, then
// negated.  The per-element Montgomery product of from_i64 made the lift
// IMAD-bound (2^27 entries: 3.1 ms, 22% of HBM); the tables make it a
// gather + adds, bound by the 32-byte writes.
template <class F>
__global__ void k_lift_luts(typename F::T* t16, typename F::T* chunks) {
  using T = typename F::T;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 65536) return;
  t16[i] = F::from_i64((int64_t)i - 32768);
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const uint64_t m = (uint64_t)i << (16 * k);
    T a = F::zero();
    a.v[0] = (uint32_t)m;
    a.v[1] = (uint32_t)(m >> 32);
    chunks[k * 65536 + i] = F::mul(a, F::r2());
  }
}
// A warp's 32 consecutive 32-byte elements stored as 64 consecutive 16-byte
// chunks, lane t writing chunks t and 32 + t (halves exchanged by shuffles):
// every store instruction fills whole 32-byte sectors (one element per lane,
// written as two 16-byte halves, leaves each sector half-written per
// instruction and triples the L2 sector writes).
ZKL_D void store_warp_fr(fr_t* dst_warp, const fr_t& v, int lane) {
  const uint4 lo = make_uint4(v.v[0], v.v[1], v.v[2], v.v[3]);
  const uint4 hi = make_uint4(v.v[4], v.v[5], v.v[6], v.v[7]);
  uint4* out = reinterpret_cast<uint4*>(dst_warp);
#pragma unroll
  for (int part = 0; part < 2; part++) {
    const int src = part * 16 + (lane >> 1);
    uint4 a, b;
    a.x = __shfl_sync(0xffffffffu, lo.x, src);
    a.y = __shfl_sync(0xffffffffu, lo.y, src);
    a.z = __shfl_sync(0xffffffffu, lo.z, src);
    a.w = __shfl_sync(0xffffffffu, lo.w, src);
    b.x = __shfl_sync(0xffffffffu, hi.x, src);
    b.y = __shfl_sync(0xffffffffu, hi.y, src);
    b.z = __shfl_sync(0xffffffffu, hi.z, src);
    b.w = __shfl_sync(0xffffffffu, hi.w, src);
    out[part * 32 + lane] = (lane & 1) ? b : a;
  }
}

template <class F>
__global__ void k_lift16_lut(typename F::T* dst, const int16_t* src, uint64_t n,
                             const typename F::T* t16) {
  using T = typename F::T;
  // four entries per thread per step: all four L2 table loads are in flight
  // before the first store; full warps store whole sectors (store_warp_fr)
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i - lane + 31 + 3 * stride < n; i += 4 * stride) {  // warp-uniform condition
    T v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) v[k] = t16[(int)src[i + k * stride] + 32768];
    if constexpr (F::kId == 0) {
#pragma unroll
      for (int k = 0; k < 4; k++) store_warp_fr(dst + (i - lane) + k * stride, v[k], lane);
    } else {
#pragma unroll
      for (int k = 0; k < 4; k++) dst[i + k * stride] = v[k];
    }
  }
  for (; i < n; i += stride) dst[i] = t16[(int)src[i] + 32768];
}
// int16 -> Fr255 Montgomery form without a table: x R mod p = m R1 - q p for
// m = |x| < 2^15 (R1 = R mod p), q = floor(m R1 / p) estimated in float64
// (off by at most one, corrected), then negated for x < 0.  16 IMAD.WIDE and
// two carry chains per entry in registers, so the kernel is bound by its 2 B
// read + 32 B write stream, not by the L2 table gathers of k_lift16_lut.
ZKL_D fr_t lift16_direct(int x) {
  const uint32_t R1[8] = {0xfffffffeu, 0x00000001u, 0x00034802u, 0x5884b7fau,
                          0xecbc4ff5u, 0x998c4fefu, 0xacc5056fu, 0x1824b159u};
  const uint32_t P[8] = {Fr255::P0, Fr255::P1, Fr255::P2, Fr255::P3,
                         Fr255::P4, Fr255::P5, Fr255::P6, Fr255::P7};
  const uint32_t m = (uint32_t)(x < 0 ? -x : x);
  const uint32_t q = (uint32_t)((double)m * 0.20826083002509044);  // R1 / p
  // t = m R1 - q p (both < 2^271; the difference is in (-p, 2p))
  uint64_t ca = 0, cb = 0;
  int64_t br = 0;
  uint32_t t[9];
#pragma unroll
  for (int k = 0; k < 8; k++) {
    ca += (uint64_t)m * R1[k];
    cb += (uint64_t)q * P[k];
    const int64_t d = (int64_t)(uint32_t)ca - (int64_t)(uint32_t)cb + br;
    t[k] = (uint32_t)d;
    br = d >> 32;  // -1, 0 (arithmetic shift)
    ca >>= 32;
    cb >>= 32;
  }
  t[8] = (uint32_t)((int64_t)ca - (int64_t)cb + br);  // 0, or all ones when negative
  fr_t r;
#pragma unroll
  for (int k = 0; k < 8; k++) r.v[k] = t[k];
  if ((int32_t)t[8] < 0) {  // q was one too large: add p
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const uint64_t v = (uint64_t)r.v[k] + P[k] + c;
      r.v[k] = (uint32_t)v;
      c = (uint32_t)(v >> 32);
    }
  } else {
    // q one too small: r >= p (r < 2p < 2^256 always fits the 8 limbs)
    bool ge = true;
#pragma unroll
    for (int k = 7; k >= 0; k--) {
      if (r.v[k] != P[k]) {
        ge = r.v[k] > P[k];
        break;
      }
    }
    if (ge) {
      int64_t b = 0;
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const int64_t v = (int64_t)r.v[k] - P[k] + b;
        r.v[k] = (uint32_t)v;
        b = v >> 32;
      }
    }
  }
  if (x < 0) {  // p - r (r != 0 for x != 0)
    int64_t b = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int64_t v = (int64_t)P[k] - r.v[k] + b;
      r.v[k] = (uint32_t)v;
      b = v >> 32;
    }
  }
  return r;
}

__global__ void k_lift16_direct(fr_t* dst, const int16_t* src, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i - lane + 31 + 3 * stride < n; i += 4 * stride) {  // warp-uniform condition
    int x[4];
#pragma unroll
    for (int k = 0; k < 4; k++) x[k] = __ldcs(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; k++) store_warp_fr(dst + (i - lane) + k * stride, lift16_direct(x[k]), lane);
  }
  for (; i < n; i += stride) dst[i] = lift16_direct(src[i]);
}

template <class F, class I>
__global__ void k_lift_chunks(typename F::T* dst, const I* src, uint64_t n,
                              const typename F::T* chunks) {
  using T = typename F::T;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t x = (int64_t)src[i];
    const uint64_t m = x < 0 ? (uint64_t)(-(x + 1)) + 1u : (uint64_t)x;
    T r = chunks[m & 0xffffu];
    if (m >> 16) {
      r = F::add(r, chunks[65536 + ((m >> 16) & 0xffffu)]);
      if (m >> 32) {
        r = F::add(r, chunks[2 * 65536 + ((m >> 32) & 0xffffu)]);
        if (m >> 48) r = F::add(r, chunks[3 * 65536 + (m >> 48)]);
      }
    }
    dst[i] = x < 0 ? F::sub(F::zero(), r) : r;
  }
}
// per-device tables, built on first use (the C-ABI is single-owner)
static std::mutex g_lut_mu;
static std::map<int, void*> g_lift_luts;
static int lift_luts_fr(const fr_t** t16, const fr_t** chunks, cudaStream_t s) {
  int dev = 0;
  ZKL_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_lut_mu);
  void*& p = g_lift_luts[dev];
  if (!p) {
    ZKL_CUDA(cudaMalloc(&p, 5 * 65536 * sizeof(fr_t)));
    fr_t* base = (fr_t*)p;
    k_lift_luts<Fr255><<<256, 256, 0, s>>>(base, base + 65536);
    ZKL_LAUNCH_CHECK();
  }
  *t16 = (const fr_t*)p;
  *chunks = (const fr_t*)p + 65536;
  return kOk;
}

template <class F>
int op_lift(void* dst, const void* src, int mtype, uint64_t n, cudaStream_t s) {
  if (!n) return kOk;
  auto* d = (typename F::T*)dst;
  unsigned g = grid_for(n, 256);
  if constexpr (F::kId == 0) {
    if (n >= 4096 && mtype >= 1 && mtype <= 3) {
      const fr_t *t16, *ch;
      int rc = lift_luts_fr(&t16, &ch, s);
      if (rc) return rc;
      switch (mtype) {
        case 1:
          if constexpr (F::kId == 0) {
            static const bool lut = getenv("ZKL_LIFT_LUT") != nullptr;
            if (!lut) {
              k_lift16_direct<<<g, 256, 0, s>>>((fr_t*)d, (const int16_t*)src, n);
              break;
            }
          }
          k_lift16_lut<F><<<g, 256, 0, s>>>(d, (const int16_t*)src, n, t16);
          break;
        case 2: k_lift_chunks<F, int32_t><<<g, 256, 0, s>>>(d, (const int32_t*)src, n, ch); break;
        default: k_lift_chunks<F, int64_t><<<g, 256, 0, s>>>(d, (const int64_t*)src, n, ch); break;
      }
      ZKL_LAUNCH_CHECK();
      return kOk;
    }
  }
  switch (mtype) {
    case 1: k_lift<F, int16_t><<<g, 256, 0, s>>>(d, (const int16_t*)src, n); break;
    case 2: k_lift<F, int32_t><<<g, 256, 0, s>>>(d, (const int32_t*)src, n); break;
    case 3: k_lift<F, int64_t><<<g, 256, 0, s>>>(d, (const int64_t*)src, n); break;
    default: set_error("lift: bad integer type %d", mtype); return kErrArg;
  }
  ZKL_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------------------
// eq table: eq[idx] = prod_j (bit_{m-1-j}(idx) ? r_j : 1 - r_j)   (mle.py:67-82)
// Two-level: eq = hi (x) lo with hi over the first mh coordinates.
template <class F>
__global__ void k_eq_direct(typename F::T* dst, PointArg<F> pt, int off, int m) {
  uint64_t n = 1ull << m;
  // two interleaved product chains (first / second half of the coordinates)
  // halve the dependent-multiply latency of this latency-bound kernel
  const int mh = m / 2;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    typename F::T a = F::one(), b = F::one();
    int j = 0;
    for (; j < mh; j++) {
      const int k = mh + j;
      const bool ba = (i >> (m - 1 - j)) & 1, bb = (i >> (m - 1 - k)) & 1;
      F::mul2(a, ba ? pt.r[off + j] : pt.omr[off + j], b, bb ? pt.r[off + k] : pt.omr[off + k],
              a, b);
    }
    if (2 * mh < m) {  // odd m: last coordinate
      const int k = m - 1;
      const bool bb = (i >> (m - 1 - k)) & 1;
      b = F::mul(b, bb ? pt.r[off + k] : pt.omr[off + k]);
    }
    dst[i] = F::mul(a, b);
  }
}
template <class F>
__global__ void k_eq_outer(typename F::T* dst, const typename F::T* hi, const typename F::T* lo,
                           int ml, uint64_t n) {
  uint64_t mask = (1ull << ml) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = F::mul(hi[i >> ml], lo[i & mask]);
}

// eq over m <= 16 coordinates with a product tree of depth ~log2(m):
// level 1 (per block, in shared memory): coordinates in pairs, 4 entries per
// pair = one product each; level 2 (per output): product of the <= 8 pair
// values as a balanced tree.  ~4 dependent Montgomery products for m = 12
// instead of m/2 in the two-chain direct form.
#ifndef ZKL_EQ_ONE_LANE
constexpr bool kEqLanes4 = true;
#else
constexpr bool kEqLanes4 = false;
#endif
template <class F>
ZKL_D void eq_tree_body(typename F::T* dst, const PointArg<F>& pt, int off, int m) {
  using T = typename F::T;
  __shared__ T grp[8][4];
  const int G = (m + 1) / 2;
  const int t = threadIdx.x;
  if (t < 4 * G) {
    const int g = t >> 2, e = t & 3;
    const int j0 = 2 * g, j1 = 2 * g + 1;
    const T a = (e >> 1) ? pt.r[off + j0] : pt.omr[off + j0];
    if (j1 < m) {
      const T b = (e & 1) ? pt.r[off + j1] : pt.omr[off + j1];
      grp[g][e] = F::mul(a, b);
    } else {
      grp[g][e] = a;  // odd m: single-coordinate group (entries 0/2 and 1/3 alias)
    }
  }
  __syncthreads();
  const uint64_t n = 1ull << m;
#ifndef ZKL_EQ_ONE_LANE
  if (G >= 3 && m >= 3) {
    // four lanes per output: lane q multiplies the pair values of groups
    // 2q and 2q + 1 (one product), then two shuffle-and-multiply steps: 3
    // single dependent products after the pair stage, instead of the
    // interleaved mul4 / mul2 / mul tree (the kernel is latency-bound)
    const uint64_t lanes = 4 * n;  // a multiple of 32 for m >= 3
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + t; l < lanes;
         l += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t i = l >> 2;
      const int q = (int)(l & 3);
      auto val = [&](int g) -> T {
        if (g >= G) return F::one();
        const int j0 = 2 * g;
        const int b0 = (int)((i >> (m - 1 - j0)) & 1);
        const int b1 = j0 + 1 < m ? (int)((i >> (m - 2 - j0)) & 1) : 0;
        return grp[g][(b0 << 1) | b1];
      };
      T x = 2 * q + 1 < G ? F::mul(val(2 * q), val(2 * q + 1)) : val(2 * q);
      x = F::mul(x, shfl_xor(x, 1));
      if (G > 4) x = F::mul(x, shfl_xor(x, 2));
      if (q == 0) dst[i] = x;
    }
    return;
  }
#endif
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + t; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    T v[8];
#pragma unroll
    for (int g = 0; g < 8; g++) {
      if (g < G) {
        const int j0 = 2 * g;
        const int b0 = (int)((i >> (m - 1 - j0)) & 1);
        const int b1 = j0 + 1 < m ? (int)((i >> (m - 2 - j0)) & 1) : 0;
        v[g] = grp[g][(b0 << 1) | b1];
      } else {
        v[g] = F::one();
      }
    }
    // balanced product tree over 8 slots (slots >= G are one)
    T a, b, c, d;
    if (G > 4) {
      F::mul4(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], a, b, c, d);
      F::mul2(a, b, c, d, a, c);
      dst[i] = F::mul(a, c);
    } else if (G > 2) {
      F::mul2(v[0], v[1], v[2], v[3], a, c);
      dst[i] = F::mul(a, c);
    } else if (G == 2) {
      dst[i] = F::mul(v[0], v[1]);
    } else {
      dst[i] = v[0];
    }
  }
}
template <class F>
__global__ void __launch_bounds__(256) k_eq_tree(typename F::T* dst, PointArg<F> pt, int off,
                                                 int m) {
  eq_tree_body<F>(dst, pt, off, m);
}
// the point read from memory the host rewrites between graph replays (mapped
// host memory: one parallel burst of 4-byte loads into shared memory, so the
// PCIe round trip is paid once per block, not per dependent read)
template <class F>
__global__ void __launch_bounds__(256) k_eq_tree_dev(typename F::T* dst, const PointArg<F>* pt,
                                                     int m) {
  __shared__ PointArg<F> sp;
  constexpr int kW = sizeof(typename F::T) / 4;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(pt);
  uint32_t* d = reinterpret_cast<uint32_t*>(&sp);
  for (int i = threadIdx.x; i < 2 * m * kW; i += blockDim.x) {
    const int w = i < m * kW ? i : kMaxPoint * kW + (i - m * kW);  // r[0..m), then omr[0..m)
    d[w] = src[w];
  }
  __syncthreads();
  eq_tree_body<F>(dst, sp, 0, m);
}
// r[0..m) and omr[0..m) of a point in mapped host memory -> device memory, by
// one block of 16-byte loads (a PCIe read per 16 bytes, once per table, not
// once per block of the table kernel)
template <class F>
__global__ void k_point_to_dev(const PointArg<F>* src, PointArg<F>* dst, int m) {
  constexpr int kV = sizeof(typename F::T) / 16 > 0 ? sizeof(typename F::T) / 16 : 1;
  const int per = (int)(m * sizeof(typename F::T) + 15) / 16;  // uint4 per array
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  constexpr int kArr = (int)(kMaxPoint * sizeof(typename F::T) / 16);  // omr offset (uint4)
  (void)kV;
  for (int i = threadIdx.x; i < 2 * per; i += blockDim.x) {
    const int w = i < per ? i : kArr + (i - per);
    d[w] = s[w];
  }
}
template <class F>
int op_eq_table_dev(void* dst, const PointArg<F>* pt_dev, int m, int slot_id, cudaStream_t s) {
  if (m < 1 || m > 16) { set_error("eq_table_dev: m=%d unsupported", m); return kErrArg; }
  if (slot_id < 0 || slot_id >= 8) { set_error("eq_table_dev: slot %d", slot_id); return kErrArg; }
  // device copies of the points, one per caller slot (tables built
  // concurrently on two streams use different slots)
  static PointArg<F>* staged = nullptr;
  if (!staged) ZKL_CUDA(cudaMalloc((void**)&staged, 8 * sizeof(PointArg<F>)));
  PointArg<F>* slot = staged + slot_id;
  k_point_to_dev<F><<<1, 64, 0, s>>>(pt_dev, slot, m);
  ZKL_LAUNCH_CHECK();
  k_eq_tree_dev<F><<<grid_for((kEqLanes4 && m >= 5 ? 4ull : 1ull) << m, 256), 256, 0, s>>>(
      (typename F::T*)dst, slot, m);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

template <class F>
int op_eq_table(void* dst, const typename F::T* point, int m, cudaStream_t s) {
  using T = typename F::T;
  if (m < 0 || m > kMaxPoint) { set_error("eq_table: m=%d unsupported", m); return kErrArg; }
  PointArg<F> pt;
  for (int j = 0; j < m; j++) {
    pt.r[j] = point[j];
    pt.omr[j] = F::sub(F::one(), point[j]);
  }
  T* out = (T*)dst;
  if (m == 0) {
    k_eq_direct<F><<<1, 32, 0, s>>>(out, pt, 0, m);
    ZKL_LAUNCH_CHECK();
    return kOk;
  }
  if (m <= 16) {
    k_eq_tree<F><<<grid_for((kEqLanes4 && m >= 5 ? 4ull : 1ull) << m, 256), 256, 0, s>>>(out, pt, 0,
                                                                                      m);
    ZKL_LAUNCH_CHECK();
    return kOk;
  }
  if (m > 32) { set_error("eq_table: 2^%d entries is beyond device memory", m); return kErrArg; }
  int mh = m / 2, ml = m - mh;
  void* ws;
  int rc = scratch_reserve(((1ull << mh) + (1ull << ml)) * sizeof(T), &ws, s);
  if (rc) return rc;
  T* hi = (T*)ws;
  T* lo = hi + (1ull << mh);
  k_eq_tree<F><<<grid_for((kEqLanes4 ? 4ull : 1ull) << mh, 256), 256, 0, s>>>(hi, pt, 0, mh);
  ZKL_LAUNCH_CHECK();
  k_eq_tree<F><<<grid_for((kEqLanes4 ? 4ull : 1ull) << ml, 256), 256, 0, s>>>(lo, pt, mh, ml);
  ZKL_LAUNCH_CHECK();
  k_eq_outer<F><<<grid_for(1ull << m, 256), 256, 0, s>>>(out, hi, lo, ml, 1ull << m);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------------------
// fold: dst[i] = src[i] + r (src[i+half] - src[i])   (mle.py:50-56)
template <class F>
__global__ void k_fold(typename F::T* dst, const typename F::T* src, uint64_t half,
                       typename F::T r) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < half;
       i += (uint64_t)gridDim.x * blockDim.x) {
    typename F::T a = src[i], b = src[i + half];
    dst[i] = F::add(a, F::mul(r, F::sub(b, a)));
  }
}
template <class F>
int op_fold(void* dst, const void* src, uint64_t half, typename F::T r, cudaStream_t s) {
  if (!half) return kOk;
  k_fold<F><<<grid_for(half, 256), 256, 0, s>>>((typename F::T*)dst,
                                                 (const typename F::T*)src, half, r);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

template <class F>
__global__ void k_axpy(typename F::T* y, const typename F::T* a, typename F::T k,
                       const typename F::T* b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    y[i] = F::add(a[i], F::mul(k, b[i]));
}
template <class F>
int op_axpy(void* y, const void* a, typename F::T k, const void* b, uint64_t n, cudaStream_t s) {
  if (!n) return kOk;
  k_axpy<F><<<grid_for(n, 256), 256, 0, s>>>((typename F::T*)y, (const typename F::T*)a, k,
                                              (const typename F::T*)b, n);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

// pointwise product dst[i] = a[i] b[i]
template <class F>
__global__ void k_mul(typename F::T* dst, const typename F::T* a, const typename F::T* b,
                      uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = F::mul(a[i], b[i]);
}
template <class F>
int op_mul(void* dst, const void* a, const void* b, uint64_t n, cudaStream_t s) {
  if (!n) return kOk;
  k_mul<F><<<grid_for(n, 256), 256, 0, s>>>((typename F::T*)dst, (const typename F::T*)a,
                                             (const typename F::T*)b, n);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

// single-block dot / sum (vectors here are <= a few 2^12 entries)
template <class F>
__global__ void k_dot(typename F::T* out, const typename F::T* a, const typename F::T* b,
                      uint64_t n) {
  using T = typename F::T;
  __shared__ T sm[32];
  T acc[1] = {F::zero()};
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x)
    acc[0] = F::add(acc[0], b ? F::mul(a[i], b[i]) : a[i]);
  block_sum<F, 1>(acc, sm);
  if (threadIdx.x == 0) *out = acc[0];
}
// Block partial sums of a[i] * b[i] over a grid (one product per thread per
// step), then one block sums the partials: a single block doing all n
// Montgomery products was issue-bound on one SM (n = 2^16: ~160 us).
template <class F>
__global__ void k_dot_partial(typename F::T* part, const typename F::T* a,
                              const typename F::T* b, uint64_t n) {
  using T = typename F::T;
  __shared__ T sm[32];
  T acc[1] = {F::zero()};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc[0] = F::add(acc[0], b ? F::mul(a[i], b[i]) : a[i]);
  block_sum<F, 1>(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
}
// partial sums of the grid-wide dot, one buffer per (device, stream): two
// streams running dots concurrently (the zkMat side stream, callers on other
// torch streams) must not share it.  Not the scratch arena, whose current
// reservation may hold the caller's output.
static std::mutex g_dot_mu;
static std::map<std::pair<int, cudaStream_t>, void*>& dot_partials() {
  static std::map<std::pair<int, cudaStream_t>, void*> m;
  return m;
}
template <class F>
int op_dot(typename F::T* out_dev, const void* a, const void* b, uint64_t n, cudaStream_t s) {
  using T = typename F::T;
  constexpr unsigned kMaxParts = 512;
  if (n <= 2048) {
    k_dot<F><<<1, 1024, 0, s>>>(out_dev, (const T*)a, (const T*)b, n);
    ZKL_LAUNCH_CHECK();
    return kOk;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  void* part;
  {
    std::lock_guard<std::mutex> lk(g_dot_mu);
    void*& slot = dot_partials()[{dev, s}];
    if (!slot) ZKL_CUDA(cudaMalloc(&slot, kMaxParts * 32));
    part = slot;
  }
  unsigned g = (unsigned)((n + 255) / 256);
  if (g > kMaxParts) g = kMaxParts;
  k_dot_partial<F><<<g, 256, 0, s>>>((T*)part, (const T*)a, (const T*)b, n);
  ZKL_LAUNCH_CHECK();
  k_dot<F><<<1, 512, 0, s>>>(out_dev, (const T*)part, nullptr, g);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

// expand: mode 0 (pad):  dst[i] = i < src_n ? (src ? src[i] : 0) + add : pad
//         mode 1 (tile): dst[i] = (src ? src[i % src_n] : 0) + add
// (lookup.py:188-202: zero-padded secret side / replicated table side)
template <class F>
__global__ void k_expand(typename F::T* dst, uint64_t dst_n, const typename F::T* src,
                         uint64_t src_n, int mode, typename F::T add, typename F::T pad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < dst_n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    typename F::T v;
    if (mode == 0) {
      v = i < src_n ? (src ? F::add(src[i], add) : add) : pad;
    } else {
      v = src ? F::add(src[i % src_n], add) : add;
    }
    dst[i] = v;
  }
}
template <class F>
int op_expand(void* dst, uint64_t dst_n, const void* src, uint64_t src_n, int mode,
              typename F::T add, typename F::T pad, cudaStream_t s) {
  if (!dst_n) return kOk;
  if (mode == 1 && src_n == 0) { set_error("expand: empty tile source"); return kErrArg; }
  k_expand<F><<<grid_for(dst_n, 256), 256, 0, s>>>((typename F::T*)dst, dst_n,
                                                    (const typename F::T*)src, src_n, mode,
                                                    add, pad);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

// dst[i] = src[idx[i]] (+ add): the secret-side logUp columns of a lookup
// whose secret entries are known table entries (idx from
// zkl_multiplicities_index), e.g. 1/(beta + s_i) = 1/(beta + t_idx(i)).
template <class F, bool ADD>
__global__ void k_gather(typename F::T* dst, const typename F::T* src, const uint32_t* idx,
                         uint64_t n, typename F::T add) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    typename F::T v = src[__ldg(idx + i)];
    if (ADD) v = F::add(v, add);
    dst[i] = v;
  }
}
template <class F>
int op_gather(void* dst, const void* src, uint64_t src_n, const uint32_t* idx, uint64_t n,
              typename F::T add, bool has_add, cudaStream_t s) {
  if (!n) return kOk;
  if (!src_n) { set_error("gather: empty source"); return kErrArg; }
  using T = typename F::T;
  if (has_add)
    k_gather<F, true><<<grid_for(n, 256), 256, 0, s>>>((T*)dst, (const T*)src, idx, n, add);
  else
    k_gather<F, false><<<grid_for(n, 256), 256, 0, s>>>((T*)dst, (const T*)src, idx, n, add);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

// u32 counts -> field
template <class F>
__global__ void k_lift_u32(typename F::T* dst, const uint32_t* src, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = F::from_u32(src[i]);
}
template <class F>
int op_lift_u32(void* dst, const uint32_t* src, uint64_t n, cudaStream_t s) {
  if (!n) return kOk;
  k_lift_u32<F><<<grid_for(n, 256), 256, 0, s>>>((typename F::T*)dst, src, n);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

template <class F>
int op_read(uint8_t* host, const void* src, uint64_t n, cudaStream_t s) {
  using T = typename F::T;
  if (!n) return kOk;
  void* ws;
  int rc = scratch_reserve(n * sizeof(T), &ws, s);
  if (rc) return rc;
  rc = op_from_mont<F>(ws, src, n, s);
  if (rc) return rc;
  ZKL_CUDA(cudaMemcpyAsync(host, ws, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  return kOk;
}

// ---------------------------------------------------------------------------
// Rescale witness (gadgets.py:563-580, quantize.py:101-104): for every wide
// entry w, q = floor((w + divisor/2) / divisor), r = w - divisor q (so r is in
// [-divisor/2, divisor/2)), resid = r * lift.  q outside [qmin, qmax] is the
// reference's RangeViolation (gadgets.py:575): the first such index and the
// count are reported and the caller raises -- a clamped quotient would break
// wide = divisor*q + r, which the verifier checks.  One pass: 8 B in, 4 B out.
template <class W>
__global__ void k_rescale_witness(const W* wide, uint64_t n, int64_t divisor, int shift,
                                  int64_t lift, int64_t qmin, int64_t qmax, int16_t* q_out,
                                  int16_t* r_out, unsigned long long* first_bad,
                                  unsigned long long* n_bad) {
  unsigned bad = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t w = (int64_t)wide[i];
    const int64_t t = w + divisor / 2;
    int64_t q;
    if (shift >= 0) {
      q = t >> shift;  // arithmetic shift = floor division by 2^shift
    } else {
      q = t / divisor;
      if ((t % divisor != 0) && (t < 0)) q -= 1;  // floor division
    }
    const int64_t r = w - divisor * q;
    if (q < qmin || q > qmax) {
      atomicMin(first_bad, (unsigned long long)i);
      bad++;
    }
    q_out[i] = (int16_t)q;
    r_out[i] = (int16_t)(r * lift);
  }
  bad = __reduce_add_sync(0xffffffffu, bad);
  if (bad && (threadIdx.x & 31) == 0) atomicAdd(n_bad, (unsigned long long)bad);
}

int op_rescale_witness(const void* wide, int wide_type, uint64_t n, int64_t divisor, int64_t lift,
                       int64_t qmin, int64_t qmax, int16_t* q_out, int16_t* r_out,
                       int64_t* first_bad, uint64_t* n_bad, cudaStream_t s) {
  *first_bad = -1;
  *n_bad = 0;
  if (divisor <= 0 || qmin < -32768 || qmax > 32767 || divisor / 2 * lift > 32768) {
    set_error("rescale_witness: quotient / residue must fit int16");
    return kErrArg;
  }
  void* ws;
  int rc = scratch_reserve(64, &ws, s);
  if (rc) return rc;
  unsigned long long* flag = (unsigned long long*)ws;
  ZKL_CUDA(cudaMemsetAsync(flag, 0xff, 8, s));
  ZKL_CUDA(cudaMemsetAsync(flag + 1, 0, 8, s));
  int shift = -1;  // divisor = 2^shift: shifts instead of 64-bit division
  if ((divisor & (divisor - 1)) == 0) {
    shift = 0;
    while ((1ll << shift) < divisor) shift++;
  }
  if (n) {
    const unsigned g = grid_for(n, 256);
    switch (wide_type) {
      case 1: k_rescale_witness<int16_t><<<g, 256, 0, s>>>((const int16_t*)wide, n, divisor, shift, lift,
                  qmin, qmax, q_out, r_out, flag, flag + 1); break;
      case 2: k_rescale_witness<int32_t><<<g, 256, 0, s>>>((const int32_t*)wide, n, divisor, shift, lift,
                  qmin, qmax, q_out, r_out, flag, flag + 1); break;
      case 3: k_rescale_witness<int64_t><<<g, 256, 0, s>>>((const int64_t*)wide, n, divisor, shift, lift,
                  qmin, qmax, q_out, r_out, flag, flag + 1); break;
      default: set_error("rescale_witness: int16/int32/int64 only"); return kErrArg;
    }
    ZKL_LAUNCH_CHECK();
  }
  void* pin;
  if ((rc = pinned_reserve(16, &pin))) return rc;
  ZKL_CUDA(cudaMemcpyAsync(pin, flag, 16, cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  unsigned long long v[2];
  memcpy(v, pin, 16);
  *n_bad = v[1];
  if (v[0] != ~0ull) {
    *first_bad = (int64_t)v[0];
    return kErrMissing;
  }
  return kOk;
}

#define ZKL_INST(F)                                                                       \
  template int op_to_mont<F>(void*, const void*, uint64_t, cudaStream_t);                 \
  template int op_from_mont<F>(void*, const void*, uint64_t, cudaStream_t);               \
  template int op_lift<F>(void*, const void*, int, uint64_t, cudaStream_t);               \
  template int op_pair_combine<F>(void*, const void*, int, const void*, int, uint64_t, F::T,  \
                                  cudaStream_t);                                             \
  template int op_eq_table<F>(void*, const F::T*, int, cudaStream_t);                     \
  template int op_fold<F>(void*, const void*, uint64_t, F::T, cudaStream_t);              \
  template int op_axpy<F>(void*, const void*, F::T, const void*, uint64_t, cudaStream_t); \
  template int op_mul<F>(void*, const void*, const void*, uint64_t, cudaStream_t);          \
  template int op_read<F>(uint8_t*, const void*, uint64_t, cudaStream_t);                 \
  template int op_dot<F>(F::T*, const void*, const void*, uint64_t, cudaStream_t);          \
  template int op_eq_table_dev<F>(void*, const PointArg<F>*, int, int, cudaStream_t);        \
  template int op_expand<F>(void*, uint64_t, const void*, uint64_t, int, F::T, F::T,        \
                            cudaStream_t);                                                  \
  template int op_lift_u32<F>(void*, const uint32_t*, uint64_t, cudaStream_t);                \
  template int op_gather<F>(void*, const void*, uint64_t, const uint32_t*, uint64_t, F::T, bool, \
                            cudaStream_t);
ZKL_INST(Fr255)
ZKL_INST(M61)

}  // namespace zkl
