// Batch inversion (Montgomery's trick, hierarchical).
//
// Reference: field.py:34-46 (batch_inverse) and lookup.py:173-174 (called on
// beta + s and beta + t).  Semantics kept: any zero input raises
// InversionOfZero naming the FIRST zero index (field.py:38-39).
//
// Level l (values v, n_l of them) is split into tiles of kTile = 256 * kCh
// elements; thread t of a tile owns elements {t + 256 j : j < kCh} (coalesced).
//   pass 1: each block multiplies its tile -> one product per block
//           (thread products, then a product tree in shared memory);
//           zero inputs are reported with atomicMin on the index.
//   the block products form level l+1; recurse until one value remains,
//   which is inverted once on the host (one Fermat exponentiation).
//   pass 2 (top-down): each block rebuilds its product tree, descends it from
//           the inverse of its block product, and back-substitutes its chunk.
// Cost ~4 mults/element, reads the input twice, writes once.
#include "ops.cuh"

namespace zkl {

constexpr int kInvThreads = 256;
constexpr int kCh = 8;
constexpr uint64_t kTile = (uint64_t)kInvThreads * kCh;

template <class F>
ZKL_D typename F::T load_plus(const typename F::T* src, uint64_t idx, uint64_t n,
                              const typename F::T& add, bool has_add, bool* is_zero) {
  if (idx >= n) { *is_zero = false; return F::one(); }
  typename F::T v = src[idx];
  if (has_add) v = F::add(v, add);
  *is_zero = F::is_zero(v);
  return v;
}

// tree[1] = root, tree[k] = tree[2k] * tree[2k+1], leaves at tree[256 + t]
template <class F>
ZKL_D void build_tree(typename F::T* tree, const typename F::T& leaf) {
  const int t = threadIdx.x;
  tree[kInvThreads + t] = leaf;
  __syncthreads();
  for (int width = kInvThreads / 2; width >= 1; width >>= 1) {
    if (t < width) tree[width + t] = F::mul(tree[2 * (width + t)], tree[2 * (width + t) + 1]);
    __syncthreads();
  }
}

template <class F>
__global__ void __launch_bounds__(kInvThreads)
    k_inv_up(const typename F::T* src, uint64_t n, typename F::T add, bool has_add,
             typename F::T* block_prod, unsigned long long* first_zero) {
  using T = typename F::T;
  __shared__ T tree[2 * kInvThreads];
  const uint64_t base = blockIdx.x * kTile;
  T prod = F::one();
#pragma unroll
  for (int j = 0; j < kCh; j++) {
    uint64_t idx = base + threadIdx.x + (uint64_t)j * kInvThreads;
    bool z;
    T v = load_plus<F>(src, idx, n, add, has_add, &z);
    if (z) atomicMin(first_zero, (unsigned long long)idx);
    prod = F::mul(prod, v);
  }
  build_tree<F>(tree, prod);
  if (threadIdx.x == 0) block_prod[blockIdx.x] = tree[1];
}

template <class F>
__global__ void __launch_bounds__(kInvThreads)
    k_inv_down(const typename F::T* src, uint64_t n, typename F::T add, bool has_add,
               const typename F::T* block_inv, typename F::T* dst) {
  using T = typename F::T;
  __shared__ T tree[2 * kInvThreads];
  __shared__ T inv[2 * kInvThreads];
  const uint64_t base = blockIdx.x * kTile;
  T v[kCh], pre[kCh];
  T prod = F::one();
#pragma unroll
  for (int j = 0; j < kCh; j++) {
    uint64_t idx = base + threadIdx.x + (uint64_t)j * kInvThreads;
    bool z;
    v[j] = load_plus<F>(src, idx, n, add, has_add, &z);
    pre[j] = prod;  // product of v[0..j-1]
    prod = F::mul(prod, v[j]);
  }
  build_tree<F>(tree, prod);
  // descend: inv[k] = 1 / tree[k]
  if (threadIdx.x == 0) inv[1] = block_inv[blockIdx.x];
  __syncthreads();
  for (int width = 1; width < kInvThreads; width <<= 1) {
    int t = threadIdx.x;
    if (t < 2 * width) {
      int node = 2 * width + t;  // child index at this depth
      int sib = node ^ 1;
      inv[node] = F::mul(inv[node >> 1], tree[sib]);
    }
    __syncthreads();
  }
  T acc = inv[kInvThreads + threadIdx.x];  // 1 / prod
#pragma unroll
  for (int j = kCh - 1; j >= 0; j--) {
    uint64_t idx = base + threadIdx.x + (uint64_t)j * kInvThreads;
    if (idx < n) dst[idx] = F::mul(acc, pre[j]);
    acc = F::mul(acc, v[j]);
  }
}

template <class F>
static typename F::T host_inverse(typename F::T a) {
  // a^(p-2) by left-to-right square and multiply (host, portable arithmetic)
  using T = typename F::T;
  T e = F::modulus();
  // e = p - 2 (p is odd and > 2: subtract from the low limb without borrow)
  uint8_t* eb = reinterpret_cast<uint8_t*>(&e);
  int borrow = 2;
  for (int i = 0; i < F::kBytes && borrow; i++) {
    int d = (int)eb[i] - borrow;
    borrow = d < 0 ? 1 : 0;
    eb[i] = (uint8_t)(d & 0xff);
  }
  T r = F::one();
  for (int bit = F::kBytes * 8 - 1; bit >= 0; bit--) {
    r = F::mul(r, r);
    if ((eb[bit >> 3] >> (bit & 7)) & 1) r = F::mul(r, a);
  }
  return r;
}

template <class F>
int op_batch_inverse(void* dst, const void* src, uint64_t n, typename F::T add, bool has_add,
                     int64_t* first_zero, cudaStream_t s) {
  using T = typename F::T;
  *first_zero = -1;
  if (!n) return kOk;
  // level sizes
  uint64_t sizes[16];
  int L = 0;
  sizes[0] = n;
  while (sizes[L] > 1) {
    sizes[L + 1] = (sizes[L] + kTile - 1) / kTile;
    L++;
    if (L >= 15) { set_error("batch_inverse: too large"); return kErrArg; }
  }
  // scratch: products per level (levels 1..L) + inverses per level (1..L) + flag
  size_t elems = 0;
  for (int l = 1; l <= L; l++) elems += 2 * sizes[l];
  void* ws;
  int rc = scratch_reserve(elems * sizeof(T) + 64, &ws, s);
  if (rc) return rc;
  T* prods[16];
  T* invs[16];
  T* cur = (T*)ws;
  for (int l = 1; l <= L; l++) {
    prods[l] = cur; cur += sizes[l];
    invs[l] = cur; cur += sizes[l];
  }
  unsigned long long* flag = (unsigned long long*)cur;
  ZKL_CUDA(cudaMemsetAsync(flag, 0xff, sizeof(unsigned long long), s));
  // upward
  const T* in = (const T*)src;
  for (int l = 0; l < L; l++) {
    k_inv_up<F><<<(unsigned)sizes[l + 1], kInvThreads, 0, s>>>(
        in, sizes[l], add, has_add && l == 0, prods[l + 1], flag);
    ZKL_LAUNCH_CHECK();
    in = prods[l + 1];
  }
  // fetch top product (or the single element if n == 1) and the zero flag
  void* pin;
  rc = pinned_reserve(sizeof(T) + 16, &pin);
  if (rc) return rc;
  const T* top_src = L ? prods[L] : (const T*)src;
  ZKL_CUDA(cudaMemcpyAsync(pin, top_src, sizeof(T), cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaMemcpyAsync((char*)pin + sizeof(T), flag, 8, cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  unsigned long long fz;
  memcpy(&fz, (char*)pin + sizeof(T), 8);
  T top;
  memcpy(&top, pin, sizeof(T));
  if (L == 0) {  // n == 1: no kernel ran
    if (has_add) top = F::add(top, add);
    if (F::is_zero(top)) { *first_zero = 0; return kErrZero; }
    T iv = host_inverse<F>(top);
    ZKL_CUDA(cudaMemcpyAsync(dst, &iv, sizeof(T), cudaMemcpyHostToDevice, s));
    ZKL_CUDA(cudaStreamSynchronize(s));
    return kOk;
  }
  if (fz != ~0ull) { *first_zero = (int64_t)fz; return kErrZero; }
  T top_inv = host_inverse<F>(top);
  memcpy(pin, &top_inv, sizeof(T));
  ZKL_CUDA(cudaMemcpyAsync(invs[L], pin, sizeof(T), cudaMemcpyHostToDevice, s));
  // downward
  for (int l = L - 1; l >= 0; l--) {
    const T* vals = l ? prods[l] : (const T*)src;
    T* out = l ? invs[l] : (T*)dst;
    k_inv_down<F><<<(unsigned)sizes[l + 1], kInvThreads, 0, s>>>(vals, sizes[l], add,
                                                                  has_add && l == 0,
                                                                  invs[l + 1], out);
    ZKL_LAUNCH_CHECK();
  }
  // keep the pinned staging buffer valid until the H2D copy has consumed it
  ZKL_CUDA(cudaStreamSynchronize(s));
  return kOk;
}

template int op_batch_inverse<Fr255>(void*, const void*, uint64_t, Fr255::T, bool, int64_t*,
                                     cudaStream_t);
template int op_batch_inverse<M61>(void*, const void*, uint64_t, M61::T, bool, int64_t*,
                                   cudaStream_t);

}  // namespace zkl
