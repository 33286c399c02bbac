// Shared device helpers: element load/store, warp/block field reductions,
// per-device scratch arena, error plumbing for the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "field.cuh"

namespace zkl {

constexpr int kSMs = 148;  // B200
constexpr unsigned kFull = 0xffffffffu;

// ---- element IO -------------------------------------------------------------
template <class F>
ZKL_D typename F::T ld(const typename F::T* p) { return *p; }
template <class F>
ZKL_D void st(typename F::T* p, const typename F::T& v) { *p = v; }

// streaming (read-once) loads: keep big sweeps from evicting reused data
ZKL_D fr_t ld_stream(const fr_t* p) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint4 a = __ldcs(q), b = __ldcs(q + 1);
  fr_t r;
  r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
  r.v[4] = b.x; r.v[5] = b.y; r.v[6] = b.z; r.v[7] = b.w;
  return r;
}
ZKL_D uint64_t ld_stream(const uint64_t* p) { return __ldcs(p); }
// L2-coherent loads (data written by other blocks of the same launch)
ZKL_D fr_t ld_cg(const fr_t* p) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint4 a = __ldcg(q), b = __ldcg(q + 1);
  fr_t r;
  r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
  r.v[4] = b.x; r.v[5] = b.y; r.v[6] = b.z; r.v[7] = b.w;
  return r;
}
ZKL_D uint64_t ld_cg(const uint64_t* p) { return __ldcg(p); }
ZKL_D unsigned ld_cg(const unsigned* p) { return __ldcg(p); }

// ---- shuffles -----------------------------------------------------------------
ZKL_D fr_t shfl_down(const fr_t& x, int off) {
  fr_t y;
#pragma unroll
  for (int i = 0; i < 8; i++) y.v[i] = __shfl_down_sync(kFull, x.v[i], off);
  return y;
}
ZKL_D uint64_t shfl_down(uint64_t x, int off) { return __shfl_down_sync(kFull, x, off); }
ZKL_D fr_t shfl_idx(const fr_t& x, int src) {
  fr_t y;
#pragma unroll
  for (int i = 0; i < 8; i++) y.v[i] = __shfl_sync(kFull, x.v[i], src);
  return y;
}
ZKL_D uint64_t shfl_idx(uint64_t x, int src) { return __shfl_sync(kFull, x, src); }
ZKL_D fr_t shfl_xor(const fr_t& x, int mask) {
  fr_t y;
#pragma unroll
  for (int i = 0; i < 8; i++) y.v[i] = __shfl_xor_sync(kFull, x.v[i], mask);
  return y;
}
ZKL_D uint64_t shfl_xor(uint64_t x, int mask) { return __shfl_xor_sync(kFull, x, mask); }

template <class F>
ZKL_D typename F::T warp_sum(typename F::T x) {
#pragma unroll
  for (int off = 16; off; off >>= 1) x = F::add(x, shfl_down(x, off));
  return x;
}

// Block-wide sum of NV field values per thread; result valid in thread 0.
// smem must hold (blockDim.x/32) * NV elements.
template <class F, int NV>
ZKL_D void block_sum(typename F::T (&v)[NV], typename F::T* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; j++) v[j] = warp_sum<F>(v[j]);
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NV; j++) smem[warp * NV + j] = v[j];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < NV; j++) v[j] = lane < nw ? smem[lane * NV + j] : F::zero();
#pragma unroll
    for (int j = 0; j < NV; j++) v[j] = warp_sum<F>(v[j]);
  }
  __syncthreads();
}

// ---- launch geometry ------------------------------------------------------------
inline unsigned grid_for(uint64_t work, unsigned block, unsigned max_per_sm = 8) {
  uint64_t g = (work + block - 1) / block;
  uint64_t cap = (uint64_t)kSMs * max_per_sm;
  if (g > cap) g = cap;
  if (g == 0) g = 1;
  return (unsigned)g;
}

// ---- host-side status ------------------------------------------------------------
enum Status : int {
  kOk = 0,
  kErrCuda = -1,
  kErrArg = -2,
  kErrZero = -3,      // inversion of zero (first index reported)
  kErrMissing = -4,   // element not in table (first index reported)
  kErrUnsupported = -5,
};

void set_error(const char* fmt, ...);
const char* get_error();

#define ZKL_CUDA(call)                                                         \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      ::zkl::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,              \
                       cudaGetErrorString(e_));                                \
      return ::zkl::kErrCuda;                                                  \
    }                                                                          \
  } while (0)

// every kernel launch is followed by exactly one ZKL_LAUNCH_CHECK, which also
// counts it (zkl_launch_count, used by bench.py's gpu_launches)
extern unsigned long long g_launches;
#define ZKL_LAUNCH_CHECK()          \
  do {                              \
    ++::zkl::g_launches;            \
    ZKL_CUDA(cudaGetLastError());   \
  } while (0)

// Per-device scratch arena (single owner, stream-ordered reuse).  Grows by
// reallocating; callers must not hold pointers across zkl_* calls.
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
  void* pinned = nullptr;  // small pinned host staging buffer
  size_t pinned_bytes = 0;
  void* fixed = nullptr;   // 4 KB device block, zeroed once: round ticket, flags
  void* work = nullptr;    // gadget-driver vectors (zkmat.cu), separate from scratch
  size_t work_bytes = 0;
};
Scratch& scratch_for_current_device();
cudaStream_t side_stream();  // per-device non-blocking stream with its own scratch arena
int scratch_reserve(size_t bytes, void** out, cudaStream_t s);
int pinned_reserve(size_t bytes, void** out);
// driver work arena (stream-ordered; grows by sync + realloc)
int work_reserve(size_t bytes, void** out, cudaStream_t s);
// changes whenever a scratch / work arena is reallocated (graph validity)
uint64_t arena_generation();
// fixed device words (zero-initialised once per device)
int fixed_words(void** out);
constexpr size_t kFixedTicket = 0;    // u32, k_round last-block ticket (self-resetting)
constexpr size_t kFixedFail = 64;     // u32, persistent-kernel failure flag
constexpr size_t kFixedPhaseTicket = 128;  // u32, persistent-kernel round ticket (self-resetting)
constexpr size_t kFixedBcast = 256;   // challenge broadcast slot (tagged words, L2)

// Host <-> device mailbox in mapped pinned memory (persistent sumcheck).
// Every payload word travels as a TAGGED 64-bit word (u32 payload | seq <<
// 32), written and read with single 8-byte accesses, so a reader knows a
// message is complete when every word carries the expected sequence number:
// no flag word and no system-scope fence on either side.
constexpr int kMbMaxOut = 18;         // raw outputs per round (paired SUM2PROD2: 18)
constexpr int kMbEvalWords = kMbMaxOut * 9;  // x 9 words (wide Fr sums)
constexpr int kMbFinalWords = 8 * 8;  // up to 8 tables x 8 words
constexpr int kMbTailWords = 3 * 64 * 8;  // host-tail tables: k x 2^h entries x 8 words
struct alignas(128) Mailbox {
  volatile uint64_t ev[kMbEvalWords];   // device -> host: round sums
  volatile uint64_t ch[8];              // host -> device: challenge (storage form)
  volatile uint64_t ch2[8];             // host -> device: a pair's second challenge
  volatile uint64_t fin[kMbFinalWords]; // device -> host: final values (storage form)
  volatile uint32_t abort;              // host -> device
  volatile uint32_t status;             // device -> host: 1 = timed out waiting
  volatile uint32_t seq;                // host-side sequence counter (not read by the device)
  volatile uint64_t tail[kMbTailWords];  // device -> host: folded tables of a host tail
};
int mailbox_for_current_device(Mailbox** host, Mailbox** dev);

// Optional CUDA-event profiler (zkl_prof_*): kernel families bracketed on
// their launching stream, with the algorithmic bytes each launch moves.
enum ProfKind { kProfMatvec = 0, kProfPhase = 1, kProfEq = 2, kProfKinds = 3 };
bool prof_on();
// returns an opaque handle (or -1 when profiling is off); close it after the launches
int prof_open(int kind, double bytes, double units, cudaStream_t s);
void prof_close(int handle, cudaStream_t s);

}  // namespace zkl
