// Hyrax row commitments on the GPU: the Pedersen multi-exponentiation of
// commit.py:87-115 (row i of a 2^n table laid out as split_shape(n) rows x
// cols -> h^{b_i} * prod_j g_j^{t[i cols + j]} mod q) in the Schnorr groups of
// group.py:64-70 (q = 96 p + 1 for BLS12-381 Fr exponents, q = 52 (2^61 - 1) +
// 1 for the test field), bit-identical group elements.
//
// Fixed-base windows: for every generator g_j (and the blinding generator)
// the key's tables hold g_j^(d 2^(8k)) for each byte position k of an exponent
// and d < 256, so g_j^v is the product of one table entry per nonzero exponent
// byte -- no squarings at commit time, every entry independent.  A row is one
// block: each thread multiplies its entries' powers into a running product,
// then a product tree in shared memory.  Arithmetic: N x 32-bit CIOS
// Montgomery products mod q (N = 9 / 3), R = 2^(32 N).
#include <cstdint>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ops.cuh"

namespace zkl {

struct QBig {  // q = 96 p + 1 (262 bits), exponents in BLS12-381 Fr (8 words)
  static constexpr int N = 9;
  static constexpr int EW = 8;
  static constexpr uint32_t nprime = 0xa0fd5c5fu;
  static ZKL_HD uint32_t q(int i) {
    const uint32_t v[9] = {0x00000061u, 0xffffffa0u, 0xff627f9fu, 0x671d811fu,
                                    0x9cb101ffu, 0x35b10303u, 0x9b0efb13u, 0x791ebf2fu,
                                    0x0000002bu};
    return v[i];
  }
  static ZKL_HD uint32_t r2(int i) {
    const uint32_t v[9] = {0x1acd90e1u, 0xb95e7af8u, 0x56b08f5fu, 0x4eef4378u,
                                     0x8ff50f41u, 0xa293c64du, 0x43075b99u, 0xa73c118eu,
                                     0x00000002u};
    return v[i];
  }
  static ZKL_HD uint32_t one(int i) {
    const uint32_t v[9] = {0xc4cbe993u, 0x355094ddu, 0x699014e2u, 0x375260dau,
                                      0xbe0430afu, 0x7cb91f0eu, 0x0a25f758u, 0x567bec75u,
                                      0x00000006u};
    return v[i];
  }
};
struct QTest {  // q = 52 (2^61 - 1) + 1 (67 bits), exponents in the test field (2 words)
  static constexpr int N = 3;
  static constexpr int EW = 2;
  static constexpr uint32_t nprime = 0xfafafafbu;
  static ZKL_HD uint32_t q(int i) {
    const uint32_t v[3] = {0xffffffcdu, 0x7fffffffu, 0x00000006u};
    return v[i];
  }
  static ZKL_HD uint32_t r2(int i) {
    const uint32_t v[3] = {0x5deaccceu, 0x19c060f2u, 0x00000002u};
    return v[i];
  }
  static ZKL_HD uint32_t one(int i) {
    const uint32_t v[3] = {0xd89d89c5u, 0x80000007u, 0x00000002u};
    return v[i];
  }
};

namespace {

// CIOS Montgomery product a b R^-1 mod q for a, b < q (t < 2q before the
// final subtraction, q < R / 4)
template <class P>
ZKL_HD void mmul(uint32_t (&r)[P::N], const uint32_t (&a)[P::N], const uint32_t (&b)[P::N]) {
  constexpr int N = P::N;
  uint32_t t[N + 2];
#pragma unroll
  for (int k = 0; k < N + 2; k++) t[k] = 0;
#pragma unroll
  for (int i = 0; i < N; i++) {
    uint64_t c = 0;
#pragma unroll
    for (int j = 0; j < N; j++) {
      const uint64_t x = (uint64_t)a[j] * b[i] + t[j] + c;
      t[j] = (uint32_t)x;
      c = x >> 32;
    }
    uint64_t x = (uint64_t)t[N] + c;
    t[N] = (uint32_t)x;
    t[N + 1] = (uint32_t)(x >> 32);
    const uint32_t m = t[0] * P::nprime;
    x = (uint64_t)m * P::q(0) + t[0];
    c = x >> 32;
#pragma unroll
    for (int j = 1; j < N; j++) {
      x = (uint64_t)m * P::q(j) + t[j] + c;
      t[j - 1] = (uint32_t)x;
      c = x >> 32;
    }
    x = (uint64_t)t[N] + c;
    t[N - 1] = (uint32_t)x;
    t[N] = t[N + 1] + (uint32_t)(x >> 32);
  }
  uint32_t d[N];
  uint64_t borrow = 0;
#pragma unroll
  for (int j = 0; j < N; j++) {
    const uint64_t y = (uint64_t)t[j] - P::q(j) - borrow;
    d[j] = (uint32_t)y;
    borrow = (y >> 63) & 1;
  }
  const bool ge = t[N] != 0 || !borrow;
#pragma unroll
  for (int j = 0; j < N; j++) r[j] = ge ? d[j] : t[j];
}

template <class P>
ZKL_D void load_el(uint32_t (&x)[P::N], const uint32_t* src) {
#pragma unroll
  for (int j = 0; j < P::N; j++) x[j] = src[j];
}
template <class P>
ZKL_D void store_el(uint32_t* dst, const uint32_t (&x)[P::N]) {
#pragma unroll
  for (int j = 0; j < P::N; j++) dst[j] = x[j];
}
template <class P>
ZKL_D void set_one(uint32_t (&x)[P::N]) {
#pragma unroll
  for (int j = 0; j < P::N; j++) x[j] = P::one(j);
}

// canonical -> Montgomery (x R^2 R^-1), in place, n elements
template <class P>
__global__ void k_q_to_mont(uint32_t* x, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t a[P::N], r2[P::N];
  load_el<P>(a, x + (size_t)i * P::N);
#pragma unroll
  for (int j = 0; j < P::N; j++) r2[j] = P::r2(j);
  mmul<P>(a, a, r2);
  store_el<P>(x + (size_t)i * P::N, a);
}

// bases[j][k] = g_j^(2^(8k)) (Montgomery), k < W: 8 squarings per step
template <class P>
__global__ void k_q_bases(const uint32_t* gens, int ngen, int W, uint32_t* bases) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ngen) return;
  uint32_t b[P::N];
  load_el<P>(b, gens + (size_t)j * P::N);
  for (int k = 0; k < W; k++) {
    store_el<P>(bases + ((size_t)j * W + k) * P::N, b);
    if (k + 1 < W)
      for (int s = 0; s < 8; s++) mmul<P>(b, b, b);
  }
}

// tables[j][k][d] = bases[j][k]^d, d < 256: thread per (j, k, hi) fills
// d = 16 hi .. 16 hi + 15 from base^(16 hi)
template <class P>
__global__ void k_q_fill(const uint32_t* bases, int ngen, int W, uint32_t* tables) {
  const uint64_t id = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (id >= (uint64_t)ngen * W * 16) return;
  const int hi = (int)(id & 15);
  const uint64_t jk = id >> 4;  // j * W + k
  uint32_t b[P::N], b16[P::N], t[P::N];
  load_el<P>(b, bases + jk * P::N);
  mmul<P>(b16, b, b);    // b^2
  mmul<P>(b16, b16, b16);  // b^4
  mmul<P>(b16, b16, b16);  // b^8
  mmul<P>(b16, b16, b16);  // b^16
  set_one<P>(t);
  for (int h = 0; h < hi; h++) mmul<P>(t, t, b16);  // b^(16 hi)
  uint32_t* out = tables + (jk * 256 + 16 * hi) * P::N;
  for (int lo = 0; lo < 16; lo++) {
    store_el<P>(out + (size_t)lo * P::N, t);
    mmul<P>(t, t, b);
  }
}

// acc *= g_j^v from generator j's table (v: EW canonical words)
template <class P>
ZKL_D void mul_power(uint32_t (&acc)[P::N], const uint32_t* table_j, const uint32_t* v) {
  constexpr int W = 4 * P::EW;
#pragma unroll 1
  for (int k = 0; k < W; k++) {
    const uint32_t d = (v[k >> 2] >> (8 * (k & 3))) & 0xffu;
    if (!d) continue;
    uint32_t e[P::N];
    load_el<P>(e, table_j + ((size_t)k * 256 + d) * P::N);
    mmul<P>(acc, acc, e);
  }
}

// one block per row: h^{b_i} prod_j g_j^{t[i cols + j]}; output canonical
template <class P>
__global__ void __launch_bounds__(256)
    k_q_commit_rows(const uint32_t* tables, int cols, const uint32_t* vals, const uint32_t* blind,
                    int blind_gen, uint32_t* out) {
  constexpr int W = 4 * P::EW;
  constexpr size_t kTab = (size_t)W * 256 * P::N;  // words per generator table
  __shared__ uint32_t red[256][P::N];
  const int row = blockIdx.x;
  uint32_t acc[P::N];
  set_one<P>(acc);
  const uint32_t* rv = vals + (size_t)row * cols * P::EW;
  for (int j = threadIdx.x; j < cols; j += blockDim.x)
    mul_power<P>(acc, tables + (size_t)j * kTab, rv + (size_t)j * P::EW);
  if (blind && threadIdx.x == blockDim.x - 1)  // the blinding generator's table
    mul_power<P>(acc, tables + (size_t)blind_gen * kTab, blind + (size_t)row * P::EW);
  store_el<P>(red[threadIdx.x], acc);
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      uint32_t o[P::N];
#pragma unroll
      for (int w = 0; w < P::N; w++) o[w] = red[threadIdx.x + s][w];
      mmul<P>(acc, acc, o);
      store_el<P>(red[threadIdx.x], acc);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    uint32_t one_raw[P::N];
#pragma unroll
    for (int w = 0; w < P::N; w++) one_raw[w] = w == 0 ? 1u : 0u;
    mmul<P>(acc, acc, one_raw);  // out of Montgomery form
    store_el<P>(out + (size_t)row * P::N, acc);
  }
}

template <class P>
int tables_impl(const uint8_t* gens_canon, int ngen, int qbytes, uint32_t* tables,
                cudaStream_t s) {
  constexpr int W = 4 * P::EW;
  std::vector<uint32_t> h((size_t)ngen * P::N, 0);
  for (int j = 0; j < ngen; j++)
    memcpy(h.data() + (size_t)j * P::N, gens_canon + (size_t)j * qbytes, qbytes);
  uint32_t *g = nullptr, *bases = nullptr;
  ZKL_CUDA(cudaMallocAsync((void**)&g, h.size() * 4, s));
  ZKL_CUDA(cudaMallocAsync((void**)&bases, (size_t)ngen * W * P::N * 4, s));
  ZKL_CUDA(cudaMemcpyAsync(g, h.data(), h.size() * 4, cudaMemcpyHostToDevice, s));
  k_q_to_mont<P><<<(ngen + 127) / 128, 128, 0, s>>>(g, ngen);
  ZKL_LAUNCH_CHECK();
  k_q_bases<P><<<(ngen + 127) / 128, 128, 0, s>>>(g, ngen, W, bases);
  ZKL_LAUNCH_CHECK();
  const uint64_t threads = (uint64_t)ngen * W * 16;
  k_q_fill<P><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(bases, ngen, W, tables);
  ZKL_LAUNCH_CHECK();
  ZKL_CUDA(cudaFreeAsync(g, s));
  ZKL_CUDA(cudaFreeAsync(bases, s));
  ZKL_CUDA(cudaStreamSynchronize(s));  // the host buffer h goes out of scope
  return kOk;
}

template <class P>
int rows_impl(const uint32_t* tables, int cols, const uint32_t* vals, const uint32_t* blind,
              int blind_gen, int rows, int qbytes, uint8_t* out_canon, cudaStream_t s) {
  uint32_t* out = nullptr;
  ZKL_CUDA(cudaMallocAsync((void**)&out, (size_t)rows * P::N * 4, s));
  k_q_commit_rows<P><<<rows, 256, 0, s>>>(tables, cols, vals, blind, blind_gen, out);
  ZKL_LAUNCH_CHECK();
  std::vector<uint32_t> h((size_t)rows * P::N);
  ZKL_CUDA(cudaMemcpyAsync(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost, s));
  ZKL_CUDA(cudaFreeAsync(out, s));
  ZKL_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < rows; i++)
    memcpy(out_canon + (size_t)i * qbytes, h.data() + (size_t)i * P::N, qbytes);
  return kOk;
}

}  // namespace

// group 0: q = 96 p + 1 (33-byte elements, Fr exponents); 1: q = 52 (2^61-1) + 1
// (9-byte elements, test-field exponents)
size_t commit_table_bytes(int group, int ngen) {
  if (group == 0) return (size_t)ngen * 4 * QBig::EW * 256 * QBig::N * 4;
  if (group == 1) return (size_t)ngen * 4 * QTest::EW * 256 * QTest::N * 4;
  return 0;
}

int op_commit_tables(int group, const uint8_t* gens_canon, int ngen, void* tables,
                     cudaStream_t s) {
  if (ngen < 1) { set_error("commit_tables: no generators"); return kErrArg; }
  if (group == 0) return tables_impl<QBig>(gens_canon, ngen, 33, (uint32_t*)tables, s);
  if (group == 1) return tables_impl<QTest>(gens_canon, ngen, 9, (uint32_t*)tables, s);
  set_error("commit_tables: unknown group %d", group);
  return kErrArg;
}

int op_commit_rows(int group, const void* tables, int cols, const void* vals, const void* blind,
                   int blind_gen, int rows, uint8_t* out_canon, cudaStream_t s) {
  if (rows < 1 || cols < 1) { set_error("commit_rows: empty table"); return kErrArg; }
  if (group == 0)
    return rows_impl<QBig>((const uint32_t*)tables, cols, (const uint32_t*)vals,
                           (const uint32_t*)blind, blind_gen, rows, 33, out_canon, s);
  if (group == 1)
    return rows_impl<QTest>((const uint32_t*)tables, cols, (const uint32_t*)vals,
                            (const uint32_t*)blind, blind_gen, rows, 9, out_canon, s);
  set_error("commit_rows: unknown group %d", group);
  return kErrArg;
}

}  // namespace zkl
