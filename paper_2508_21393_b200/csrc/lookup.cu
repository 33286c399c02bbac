// logUp multiplicities: m_j = #{i : s_i == t_j}.
//
// Reference: lookup.py:91-99 (compute_multiplicities).  Semantics kept:
//   * duplicate table values count toward their LAST index (the reference
//     builds {value: j} in order, later j overwrite earlier ones);
//   * a secret value absent from the table raises ElementNotInTable with
//     the FIRST offending index.
// Device design: open-addressing hash table over table indices (2x load),
// built with atomicCAS / atomicMax (duplicates keep the largest index), then
// one probe per secret entry with atomicAdd on the counts and atomicMin on
// the first miss.  Optionally each secret entry's table index is written
// out (0xffffffff for a miss), which lets the lookup prover gather the
// secret-side columns from the table side instead of inverting d entries.
#include "ops.cuh"

namespace zkl {

ZKL_D uint32_t fmix32(uint32_t h) {
  h ^= h >> 16; h *= 0x85ebca6bu;
  h ^= h >> 13; h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}
ZKL_D uint32_t hash_elem(const fr_t& v) {
  uint32_t h = v.v[0] ^ (v.v[1] * 0x9e3779b1u) ^ (v.v[2] * 0x7feb352du) ^ (v.v[7] * 0x846ca68bu);
  return fmix32(h);
}
ZKL_D uint32_t hash_elem(uint64_t v) { return fmix32((uint32_t)v ^ (uint32_t)(v >> 32) * 0x9e3779b1u); }

constexpr uint32_t kEmpty = 0xffffffffu;

template <class F>
__global__ void k_ht_insert(const typename F::T* table, uint32_t n, uint32_t* slots,
                            uint32_t mask, unsigned* dup) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    typename F::T v = table[j];
    uint32_t h = hash_elem(v) & mask;
    while (true) {
      uint32_t old = atomicCAS(&slots[h], kEmpty, j);
      if (old == kEmpty) break;
      if (F::eq(table[old], v)) {  // duplicate value: keep the last index
        atomicMax(&slots[h], j);
        if (dup) atomicOr(dup, 1u);
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

// Count one warp's hits.  Equal hits are merged with __match_any_sync (one
// atomicAdd per distinct bin); a warp whose 32 hits share one bin keeps a
// running count instead, flushed when its bin changes -- the zero padding of
// a lookup (millions of queries on one bin) would otherwise serialise on one
// counter.
ZKL_D void count_hit(uint32_t hit, uint32_t* counts, uint32_t& run_bin, uint32_t& run_cnt) {
  const unsigned peers = __match_any_sync(kFull, hit);
  if (peers == kFull) {
    if (hit == kEmpty) return;  // no lane hit (tail of the range, or all missed)
    if (hit == run_bin) {
      run_cnt += 32;
    } else {
      if (run_cnt && (threadIdx.x & 31) == 0) atomicAdd(&counts[run_bin], run_cnt);
      run_bin = hit;
      run_cnt = 32;
    }
    return;
  }
  const int leader = __ffs(peers) - 1;
  if (hit != kEmpty && (threadIdx.x & 31) == leader) atomicAdd(&counts[hit], __popc(peers));
}

// One probe per secret entry; equal hits inside a warp are merged with
// __match_any_sync so each distinct table index takes ONE atomicAdd per warp
// (skewed inputs -- e.g. the zero padding of a lookup, or activations
// concentrated near 0 -- would otherwise serialise on a few counters).
template <class F>
__global__ void k_ht_count(const typename F::T* secret, uint64_t d, const typename F::T* table,
                           const uint32_t* slots, uint32_t mask, uint32_t* counts,
                           unsigned long long* first_miss, uint32_t* index_out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t run_bin = kEmpty, run_cnt = 0;  // whole-warp hits on one bin, summed locally
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < d; base += stride) {
    const uint64_t i = base + threadIdx.x;
    uint32_t hit = kEmpty;
    if (i < d) {
      const typename F::T v = ld_stream(secret + i);
      uint32_t h = hash_elem(v) & mask;
      while (true) {
        const uint32_t e = __ldg(slots + h);
        if (e == kEmpty) { atomicMin(first_miss, (unsigned long long)i); break; }
        if (F::eq(table[e], v)) { hit = e; break; }
        h = (h + 1) & mask;
      }
    }
    if (index_out != nullptr && i < d) index_out[i] = hit;
    count_hit(hit, counts, run_bin, run_cnt);
  }
  if (run_cnt && (threadIdx.x & 31) == 0) atomicAdd(&counts[run_bin], run_cnt);
}

template <class F>
int op_multiplicities(const void* secret, uint64_t d, const void* table, uint64_t n,
                      uint32_t* counts, int64_t* first_miss, cudaStream_t s,
                      uint32_t* index_out) {
  using T = typename F::T;
  *first_miss = -1;
  if (n == 0 || n > (1ull << 31)) { set_error("multiplicities: bad table size"); return kErrArg; }
  uint64_t cap = 1;
  while (cap < 2 * n) cap <<= 1;
  void* ws;
  int rc = scratch_reserve(cap * 4 + 64, &ws, s);
  if (rc) return rc;
  uint32_t* slots = (uint32_t*)ws;
  unsigned long long* flag = (unsigned long long*)((char*)ws + cap * 4);
  ZKL_CUDA(cudaMemsetAsync(slots, 0xff, cap * 4, s));
  ZKL_CUDA(cudaMemsetAsync(flag, 0xff, 8, s));
  ZKL_CUDA(cudaMemsetAsync(counts, 0, n * 4, s));
  k_ht_insert<F><<<grid_for(n, 256), 256, 0, s>>>((const T*)table, (uint32_t)n, slots,
                                                   (uint32_t)(cap - 1), nullptr);
  ZKL_LAUNCH_CHECK();
  if (d) {
    k_ht_count<F><<<grid_for(d, 256), 256, 0, s>>>((const T*)secret, d, (const T*)table, slots,
                                                    (uint32_t)(cap - 1), counts, flag, index_out);
    ZKL_LAUNCH_CHECK();
  }
  unsigned long long fm;
  void* pin;
  rc = pinned_reserve(16, &pin);
  if (rc) return rc;
  ZKL_CUDA(cudaMemcpyAsync(pin, flag, 8, cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  memcpy(&fm, pin, 8);
  if (fm != ~0ull) { *first_miss = (int64_t)fm; return kErrMissing; }
  return kOk;
}

// Pair lookups (gadgets.py:679-688) whose table x column is the consecutive
// range x0 .. x0+n-1 (tables.py:142-152): a query (x_i, y_i) with
// 0 <= x_i - x0 < n and y_i == table_y[x_i - x0] has s_i = t_(x_i - x0)
// exactly, so its bin comes from two small integer loads instead of a hash
// probe on the 32-byte combined value.  Every other query takes the hash
// probe on s_i (identical semantics: a miss is ElementNotInTable).  Used
// only when the combined table has no duplicate values (checked here with
// the hash insert; the reference maps duplicates to the last index).
template <class F, class TX, class TY>
__global__ void k_pair_count(const TX* xs, const TY* ys, uint64_t d, int64_t x0,
                             const int32_t* ty, uint32_t n, const typename F::T* secret,
                             const typename F::T* table, const uint32_t* slots, uint32_t mask,
                             uint32_t* counts, unsigned long long* first_miss,
                             uint32_t* index_out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t run_bin = kEmpty, run_cnt = 0;  // whole-warp hits on one bin, summed locally
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < d; base += stride) {
    const uint64_t i = base + threadIdx.x;
    uint32_t hit = kEmpty;
    if (i < d) {
      const int64_t xi = (int64_t)xs[i], yi = (int64_t)ys[i];
      const int64_t idx = xi - x0;
      if (idx >= 0 && idx < (int64_t)n && (int64_t)__ldg(ty + idx) == yi) {
        hit = (uint32_t)idx;
      } else if (secret == nullptr) {  // integer-only pass: the caller reruns with the values
        atomicMin(first_miss, (unsigned long long)i);
      } else {
        const typename F::T v = secret[i];
        uint32_t h = hash_elem(v) & mask;
        while (true) {
          const uint32_t e = __ldg(slots + h);
          if (e == kEmpty) { atomicMin(first_miss, (unsigned long long)i); break; }
          if (F::eq(table[e], v)) { hit = e; break; }
          h = (h + 1) & mask;
        }
      }
      if (index_out) index_out[i] = hit;
    }
    count_hit(hit, counts, run_bin, run_cnt);
  }
  if (run_cnt && (threadIdx.x & 31) == 0) atomicAdd(&counts[run_bin], run_cnt);
}

template <class F>
int op_pair_multiplicities(const void* x, int xt, const void* y, int yt, uint64_t d, int64_t x0,
                           const int32_t* ty, const void* secret, const void* table, uint64_t n,
                           uint32_t* counts, uint32_t* index_out, int64_t* first_miss,
                           cudaStream_t s) {
  using T = typename F::T;
  *first_miss = -1;
  if (n == 0 || n > (1ull << 31)) { set_error("pair multiplicities: bad table size"); return kErrArg; }
  uint64_t cap = 1;
  while (cap < 2 * n) cap <<= 1;
  void* ws;
  int rc = scratch_reserve(cap * 4 + 64, &ws, s);
  if (rc) return rc;
  uint32_t* slots = (uint32_t*)ws;
  unsigned long long* flag = (unsigned long long*)((char*)ws + cap * 4);
  unsigned* dup = (unsigned*)((char*)ws + cap * 4 + 8);
  ZKL_CUDA(cudaMemsetAsync(slots, 0xff, cap * 4, s));
  ZKL_CUDA(cudaMemsetAsync(flag, 0xff, 8, s));
  ZKL_CUDA(cudaMemsetAsync(dup, 0, 4, s));
  ZKL_CUDA(cudaMemsetAsync(counts, 0, n * 4, s));
  k_ht_insert<F><<<grid_for(n, 256), 256, 0, s>>>((const T*)table, (uint32_t)n, slots,
                                                   (uint32_t)(cap - 1), dup);
  ZKL_LAUNCH_CHECK();
  void* pin;
  if ((rc = pinned_reserve(16, &pin))) return rc;
  ZKL_CUDA(cudaMemcpyAsync(pin, dup, 4, cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  unsigned has_dup;
  memcpy(&has_dup, pin, 4);
  if (has_dup) return kErrUnsupported;  // caller takes the hash path
  if (d) {
    const unsigned g = grid_for(d, 256);
    const T* sec = (const T*)secret;
    const T* tab = (const T*)table;
    const uint32_t m = (uint32_t)(cap - 1);
#define ZKL_PC(TX, TY)                                                                         \
  k_pair_count<F, TX, TY><<<g, 256, 0, s>>>((const TX*)x, (const TY*)y, d, x0, ty, (uint32_t)n, \
                                            sec, tab, slots, m, counts, flag, index_out)
    if (xt == 1 && yt == 1) ZKL_PC(int16_t, int16_t);
    else if (xt == 1 && yt == 2) ZKL_PC(int16_t, int32_t);
    else if (xt == 2 && yt == 1) ZKL_PC(int32_t, int16_t);
    else if (xt == 2 && yt == 2) ZKL_PC(int32_t, int32_t);
    else { set_error("pair multiplicities: int16/int32 columns only"); return kErrUnsupported; }
#undef ZKL_PC
    ZKL_LAUNCH_CHECK();
  }
  unsigned long long fm;
  ZKL_CUDA(cudaMemcpyAsync(pin, flag, 8, cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  memcpy(&fm, pin, 8);
  if (fm != ~0ull) { *first_miss = (int64_t)fm; return kErrMissing; }
  return kOk;
}
// Single-column lookups against a table that IS the consecutive integer
// range x0 .. x0+n-1 (quant_range / residue_range, tables.py:109-117): a
// query's bin is its offset, and a query outside the range is in no table
// entry, so no field value is needed at all (the secret is never lifted).
// Small tables (n <= kRangeSmemBins) count in shared memory and flush once per
// block: the 2^12-entry residue table otherwise serialises 2^27 global
// atomics on 4096 counters.
constexpr uint32_t kRangeSmemBins = 12288;  // 48 KB of uint32 counters

template <class TX, bool SMEM>
__global__ void __launch_bounds__(256) k_range_count(const TX* xs, uint64_t d, int64_t x0,
                                                     uint32_t n, uint32_t* counts,
                                                     unsigned long long* first_miss,
                                                     uint32_t* index_out) {
  extern __shared__ uint32_t sh_bins[];
  if constexpr (SMEM) {
    for (uint32_t b = threadIdx.x; b < n; b += blockDim.x) sh_bins[b] = 0;
    __syncthreads();
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t run_bin = kEmpty, run_cnt = 0;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < d; base += stride) {
    const uint64_t i = base + threadIdx.x;
    uint32_t hit = kEmpty;
    if (i < d) {
      const int64_t idx = (int64_t)xs[i] - x0;
      if (idx >= 0 && idx < (int64_t)n) hit = (uint32_t)idx;
      else atomicMin(first_miss, (unsigned long long)i);
      if (index_out) index_out[i] = hit;
    }
    if constexpr (SMEM) {
      if (hit != kEmpty) atomicAdd(&sh_bins[hit], 1u);
    } else {
      count_hit(hit, counts, run_bin, run_cnt);
    }
  }
  if constexpr (SMEM) {
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < n; b += blockDim.x)
      if (sh_bins[b]) atomicAdd(&counts[b], sh_bins[b]);
  } else {
    if (run_cnt && (threadIdx.x & 31) == 0) atomicAdd(&counts[run_bin], run_cnt);
  }
}

// Range tables up to 2^16 entries (quant_range is exactly 2^16): per-block
// 16-bit bins in shared memory, two per 32-bit word (128 KB for 2^16 bins),
// so every count is a shared-memory atomic and each block flushes its n bins
// once.  A half-word that reaches 0x8000 is moved to the global counter by
// the one thread that saw it get there (atomicAdd returns the old value); the
// other threads can add at most blockDim more before that subtraction lands,
// so a half never carries into its neighbour.  Each thread reads 8 int16
// entries per 16-byte load and writes their 8 indices with two 16-byte
// stores: 2 B in + 4 B out per query, coalesced.
constexpr uint32_t kRange16Threads = 1024;

__device__ __forceinline__ void bin16_add(uint32_t* words, uint32_t* counts, uint32_t b) {
  const uint32_t sh = (b & 1) * 16;
  const uint32_t old = atomicAdd(&words[b >> 1], 1u << sh);
  if (((old >> sh) & 0xffffu) == 0x7fffu) {  // this add made the half 0x8000
    atomicSub(&words[b >> 1], 0x8000u << sh);
    atomicAdd(&counts[b], 0x8000u);
  }
}

__global__ void __launch_bounds__(kRange16Threads)
    k_range_count16(const int16_t* xs, uint64_t d, int32_t x0, uint32_t n, uint32_t* counts,
                    unsigned long long* first_miss, uint32_t* index_out) {
  extern __shared__ uint32_t words[];  // ceil(n / 2) words
  const uint32_t nw = (n + 1) / 2;
  for (uint32_t w = threadIdx.x; w < nw; w += blockDim.x) words[w] = 0;
  __syncthreads();
  const uint64_t nvec = d / 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint4* xv = reinterpret_cast<const uint4*>(xs);
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const uint4 raw = __ldcs(xv + v);
    const uint32_t w4[4] = {raw.x, raw.y, raw.z, raw.w};
    uint32_t idx[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int32_t val = (int32_t)(int16_t)(w4[k >> 1] >> (16 * (k & 1)));
      const int32_t o = val - x0;
      if (o >= 0 && o < (int32_t)n) {
        idx[k] = (uint32_t)o;
        bin16_add(words, counts, (uint32_t)o);
      } else {
        idx[k] = kEmpty;
        atomicMin(first_miss, (unsigned long long)(8 * v + k));
      }
    }
    if (index_out) {
      uint4* out = reinterpret_cast<uint4*>(index_out + 8 * v);
      __stcs(out, make_uint4(idx[0], idx[1], idx[2], idx[3]));
      __stcs(out + 1, make_uint4(idx[4], idx[5], idx[6], idx[7]));
    }
  }
  // the d % 8 tail (block 0)
  if (blockIdx.x == 0 && threadIdx.x < d - 8 * nvec) {
    const uint64_t i = 8 * nvec + threadIdx.x;
    const int32_t o = (int32_t)xs[i] - x0;
    uint32_t hit = kEmpty;
    if (o >= 0 && o < (int32_t)n) {
      hit = (uint32_t)o;
      bin16_add(words, counts, hit);
    } else {
      atomicMin(first_miss, (unsigned long long)i);
    }
    if (index_out) index_out[i] = hit;
  }
  __syncthreads();
  for (uint32_t w = threadIdx.x; w < nw; w += blockDim.x) {
    const uint32_t c = words[w];
    if (c & 0xffffu) atomicAdd(&counts[2 * w], c & 0xffffu);
    if ((c >> 16) && 2 * w + 1 < n) atomicAdd(&counts[2 * w + 1], c >> 16);
  }
}

int op_range_multiplicities(const void* x, int xt, uint64_t d, int64_t x0, uint64_t n,
                            uint32_t* counts, uint32_t* index_out, int64_t* first_miss,
                            cudaStream_t s) {
  *first_miss = -1;
  if (n == 0 || n > (1ull << 31)) { set_error("range multiplicities: bad table size"); return kErrArg; }
  void* ws;
  int rc = scratch_reserve(64, &ws, s);
  if (rc) return rc;
  unsigned long long* flag = (unsigned long long*)ws;
  ZKL_CUDA(cudaMemsetAsync(flag, 0xff, 8, s));
  ZKL_CUDA(cudaMemsetAsync(counts, 0, n * 4, s));
  // int16 queries against a range of <= 2^16 entries (every rescale's
  // quant_range lookup): the vectorised 16-bit-bin kernel; its 16-byte loads
  // need an aligned column
  if (d && xt == 1 && n <= 65536 && n > kRangeSmemBins && x0 >= INT32_MIN &&
      x0 <= INT32_MAX && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      (!index_out || (reinterpret_cast<uintptr_t>(index_out) & 15) == 0)) {
    const size_t sb = ((n + 1) / 2) * 4;
    static bool attr = false;
    if (!attr) {
      ZKL_CUDA(cudaFuncSetAttribute(k_range_count16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    128 * 1024));
      attr = true;
    }
    const unsigned per_sm = sb <= 64 * 1024 ? 2 : 1;
    const unsigned g = grid_for((d + 7) / 8, kRange16Threads, per_sm);
    k_range_count16<<<g, kRange16Threads, sb, s>>>((const int16_t*)x, d, (int32_t)x0,
                                                    (uint32_t)n, counts, flag, index_out);
    ZKL_LAUNCH_CHECK();
  } else if (d) {
    const bool smem = n <= kRangeSmemBins;
    // shared-memory bins: a few blocks per SM, each flushes n counters once
    const unsigned g = smem ? grid_for(d, 256, 2) : grid_for(d, 256);
    const size_t sb = smem ? n * 4 : 0;
#define ZKL_RC(TX)                                                                          \
  (smem ? k_range_count<TX, true><<<g, 256, sb, s>>>((const TX*)x, d, x0, (uint32_t)n, counts, \
                                                     flag, index_out)                       \
        : k_range_count<TX, false><<<g, 256, 0, s>>>((const TX*)x, d, x0, (uint32_t)n, counts, \
                                                     flag, index_out))
    if (xt == 1) ZKL_RC(int16_t);
    else if (xt == 2) ZKL_RC(int32_t);
    else if (xt == 3) ZKL_RC(int64_t);
    else { set_error("range multiplicities: int16/int32/int64 columns only"); return kErrArg; }
#undef ZKL_RC
    ZKL_LAUNCH_CHECK();
  }
  void* pin;
  if ((rc = pinned_reserve(16, &pin))) return rc;
  unsigned long long fm;
  ZKL_CUDA(cudaMemcpyAsync(pin, flag, 8, cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  memcpy(&fm, pin, 8);
  if (fm != ~0ull) { *first_miss = (int64_t)fm; return kErrMissing; }
  return kOk;
}

template int op_pair_multiplicities<Fr255>(const void*, int, const void*, int, uint64_t, int64_t,
                                           const int32_t*, const void*, const void*, uint64_t,
                                           uint32_t*, uint32_t*, int64_t*, cudaStream_t);
template int op_pair_multiplicities<M61>(const void*, int, const void*, int, uint64_t, int64_t,
                                         const int32_t*, const void*, const void*, uint64_t,
                                         uint32_t*, uint32_t*, int64_t*, cudaStream_t);

template int op_multiplicities<Fr255>(const void*, uint64_t, const void*, uint64_t, uint32_t*,
                                      int64_t*, cudaStream_t, uint32_t*);
template int op_multiplicities<M61>(const void*, uint64_t, const void*, uint64_t, uint32_t*,
                                    int64_t*, cudaStream_t, uint32_t*);

}  // namespace zkl
