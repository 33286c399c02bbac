// Montgomery-multiply throughput on sm_100a: the library's CIOS (mad.lo/hi
// carry chains, IMAD.HI at half rate) against a CIOS whose limb products are
// full-rate 64-bit IMAD.WIDE.U32 (even/odd split: the even-limb products of
// one row tile the accumulator without overlap, the odd ones likewise at a
// 32-bit offset, so a row is two add-with-carry chains).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/mont_bench tools/mont_bench.cu
//   /tmp/mont_bench [blocks_per_sm] [iters]
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2508_21393_b200/csrc/field.cuh"

using namespace zkl;
using T = fr_t;

// x[0..8] += (w[0..7]) with the carry out of word 7 added into x[8]
#define ACC8(x0, x1, x2, x3, x4, x5, x6, x7, x8, w0, w1, w2, w3, w4, w5, w6, w7)            \
  asm("add.cc.u32 %0, %0, %9;\n\taddc.cc.u32 %1, %1, %10;\n\taddc.cc.u32 %2, %2, %11;\n\t"  \
      "addc.cc.u32 %3, %3, %12;\n\taddc.cc.u32 %4, %4, %13;\n\taddc.cc.u32 %5, %5, %14;\n\t" \
      "addc.cc.u32 %6, %6, %15;\n\taddc.cc.u32 %7, %7, %16;\n\taddc.u32 %8, %8, 0;"          \
      : "+r"(x0), "+r"(x1), "+r"(x2), "+r"(x3), "+r"(x4), "+r"(x5), "+r"(x6), "+r"(x7),     \
        "+r"(x8)                                                                            \
      : "r"(w0), "r"(w1), "r"(w2), "r"(w3), "r"(w4), "r"(w5), "r"(w6), "r"(w7))
// x[0..7] += (w[0..7]), last word without carry out
#define ACC8N(x0, x1, x2, x3, x4, x5, x6, x7, w0, w1, w2, w3, w4, w5, w6, w7)                \
  asm("add.cc.u32 %0, %0, %8;\n\taddc.cc.u32 %1, %1, %9;\n\taddc.cc.u32 %2, %2, %10;\n\t"   \
      "addc.cc.u32 %3, %3, %11;\n\taddc.cc.u32 %4, %4, %12;\n\taddc.cc.u32 %5, %5, %13;\n\t" \
      "addc.cc.u32 %6, %6, %14;\n\taddc.u32 %7, %7, %15;"                                    \
      : "+r"(x0), "+r"(x1), "+r"(x2), "+r"(x3), "+r"(x4), "+r"(x5), "+r"(x6), "+r"(x7)      \
      : "r"(w0), "r"(w1), "r"(w2), "r"(w3), "r"(w4), "r"(w5), "r"(w6), "r"(w7))

#define LO(x) ((uint32_t)(x))
#define HI(x) ((uint32_t)((x) >> 32))

// one CIOS step with wide products; t < 2p before and after (t[8] = 0)
__device__ __forceinline__ void wide_step(uint32_t t[9], const T& a, uint32_t bi) {
  const uint64_t e0 = (uint64_t)a.v[0] * bi, e2 = (uint64_t)a.v[2] * bi,
                 e4 = (uint64_t)a.v[4] * bi, e6 = (uint64_t)a.v[6] * bi;
  const uint64_t o1 = (uint64_t)a.v[1] * bi, o3 = (uint64_t)a.v[3] * bi,
                 o5 = (uint64_t)a.v[5] * bi, o7 = (uint64_t)a.v[7] * bi;
  ACC8(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], LO(e0), HI(e0), LO(e2), HI(e2),
       LO(e4), HI(e4), LO(e6), HI(e6));
  ACC8N(t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], LO(o1), HI(o1), LO(o3), HI(o3), LO(o5),
        HI(o5), LO(o7), HI(o7));
  const uint32_t m = 0u - t[0];  // n' = -1 mod 2^32 (p0 = 1)
  const uint64_t f2 = (uint64_t)m * Fr255::P2, f4 = (uint64_t)m * Fr255::P4,
                 f6 = (uint64_t)m * Fr255::P6;
  const uint64_t g1 = (uint64_t)m * Fr255::P1, g3 = (uint64_t)m * Fr255::P3,
                 g5 = (uint64_t)m * Fr255::P5, g7 = (uint64_t)m * Fr255::P7;
  ACC8(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], m, 0u, LO(f2), HI(f2), LO(f4),
       HI(f4), LO(f6), HI(f6));
  ACC8N(t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], LO(g1), HI(g1), LO(g3), HI(g3), LO(g5),
        HI(g5), LO(g7), HI(g7));
#pragma unroll
  for (int j = 0; j < 8; j++) t[j] = t[j + 1];
  t[8] = 0;
}

template <int UNROLL>
__device__ __forceinline__ T wide_mul_inl(const T& a, T b) {
  uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if constexpr (UNROLL == 8) {
#pragma unroll
    for (int i = 0; i < 8; i++) wide_step(t, a, b.v[i]);
  } else if constexpr (UNROLL == 2 || UNROLL == 4) {
#pragma unroll 1
    for (int i = 0; i < 8; i += UNROLL) {
#pragma unroll
      for (int k = 0; k < UNROLL; k++) wide_step(t, a, b.v[k]);
      T c = b;
#pragma unroll
      for (int k = 0; k < 8; k++) b.v[k] = c.v[(k + UNROLL) & 7];
    }
  } else {
#pragma unroll 1
    for (int i = 0; i < 8; i++) {
      wide_step(t, a, b.v[0]);
      const uint32_t x = b.v[0];
#pragma unroll
      for (int k = 0; k < 7; k++) b.v[k] = b.v[k + 1];
      b.v[7] = x;
    }
  }
  T r;
#pragma unroll
  for (int i = 0; i < 8; i++) r.v[i] = t[i];
  return Fr255::reduce_once(r);
}

struct Tri {
  T x, y, z;
};

// variant 0: library mul3; 1: wide rolled; 2: wide unrolled; 3: library unrolled
template <int V>
__device__ __noinline__ Tri mul3v(T a0, T b0, T a1, T b1, T a2, T b2) {
  Tri q;
  if constexpr (V == 0) {
    Fr255::mul3(a0, b0, a1, b1, a2, b2, q.x, q.y, q.z);
  } else if constexpr (V == 1 || V == 2 || V >= 4) {
    constexpr int U = V == 2 ? 8 : V == 4 ? 2 : V == 5 ? 4 : 1;
    q.x = wide_mul_inl<U>(a0, b0);
    q.y = wide_mul_inl<U>(a1, b1);
    q.z = wide_mul_inl<U>(a2, b2);
  } else {
#ifdef __CUDA_ARCH__
    uint32_t t[9] = {0}, u[9] = {0}, w[9] = {0};
#pragma unroll
    for (int i = 0; i < 8; i++) {
      Fr255::cios_step(t, a0, b0.v[i]);
      Fr255::cios_step(u, a1, b1.v[i]);
      Fr255::cios_step(w, a2, b2.v[i]);
    }
    for (int i = 0; i < 8; i++) { q.x.v[i] = t[i]; q.y.v[i] = u[i]; q.z.v[i] = w[i]; }
    q.x = Fr255::reduce_once(q.x);
    q.y = Fr255::reduce_once(q.y);
    q.z = Fr255::reduce_once(q.z);
#endif
  }
  return q;
}

template <int V>
__global__ void k_bench(T* out, const T* in, int iters) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  T x = in[3 * i], y = in[3 * i + 1], z = in[3 * i + 2];
  const T k = in[0];
  for (int it = 0; it < iters; it++) {
    Tri q = mul3v<V>(x, k, y, k, z, k);
    x = q.x;
    y = q.y;
    z = q.z;
  }
  out[3 * i] = x;
  out[3 * i + 1] = y;
  out[3 * i + 2] = z;
}

constexpr int NV = 6;

int main(int argc, char** argv) {
  const int bps = argc > 1 ? atoi(argv[1]) : 2;
  const int iters = argc > 2 ? atoi(argv[2]) : 2000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * bps, n = blocks * threads;
  T* h = (T*)malloc(sizeof(T) * 3 * n);
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < 3 * n; i++)
    for (int w = 0; w < 8; w++) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i].v[w] = (uint32_t)s;
    }
  for (int i = 0; i < 3 * n; i++) h[i].v[7] &= 0x3fffffff;  // < p
  T *din, *dout;
  cudaMalloc(&din, sizeof(T) * 3 * n);
  cudaMalloc(&dout, sizeof(T) * 3 * n * NV);
  cudaMemcpy(din, h, sizeof(T) * 3 * n, cudaMemcpyHostToDevice);
  void (*ks[NV])(T*, const T*, int) = {k_bench<0>, k_bench<1>, k_bench<2>,
                                       k_bench<3>, k_bench<4>, k_bench<5>};
  const char* names[NV] = {"lib mul3 (rolled lo/hi)", "wide rolled", "wide unrolled",
                           "lib unrolled", "wide unroll 2", "wide unroll 4"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 0; v < NV; v++) {
    ks[v]<<<blocks, threads>>>(dout + 3 * n * v, din, 10);
    cudaEventRecord(e0);
    ks[v]<<<blocks, threads>>>(dout + 3 * n * v, din, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double prods = 3.0 * n * iters;
    int regs = 0;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, ks[v]);
    regs = fa.numRegs;
    printf("%-26s %8.3f ms  %.3e products/s  regs %d  err %s\n", names[v], ms, prods / (ms * 1e-3),
           regs, cudaGetErrorString(cudaGetLastError()));
  }
  T* o = (T*)malloc(sizeof(T) * 3 * n * NV);
  cudaMemcpy(o, dout, sizeof(T) * 3 * n * NV, cudaMemcpyDeviceToHost);
  for (int v = 1; v < NV; v++)
    printf("variant %d matches lib: %s\n", v,
           memcmp(o, o + 3 * n * v, sizeof(T) * 3 * n) == 0 ? "yes" : "NO");
  return 0;
}
