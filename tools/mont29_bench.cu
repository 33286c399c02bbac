// 9 x 29-bit unsaturated Montgomery product (tools/mont29.cuh) against the
// library's 32-bit CIOS: host correctness check (no GPU needed, "check"),
// then device throughput (3 independent products per call) and latency
// (one dependent chain per warp).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/m29 tools/mont29_bench.cu
//   /tmp/m29 check | /tmp/m29 [blocks_per_sm] [iters]
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2508_21393_b200/csrc/field.cuh"
#include "mont29.cuh"

using namespace zkl;
using T = fr_t;

ZKL_HD T mul29(const T& a, const T& b) {
  T r;
  m29::mul(a.v, b.v, r.v);
  return Fr255::reduce_once(r);
}

struct Tri {
  T x, y, z;
};

template <int V>
__device__ __noinline__ Tri mul3v(T a0, T b0, T a1, T b1, T a2, T b2) {
  Tri q;
  if constexpr (V == 0) {
    Fr255::mul3(a0, b0, a1, b1, a2, b2, q.x, q.y, q.z);
  } else {
    q.x = mul29(a0, b0);
    q.y = mul29(a1, b1);
    q.z = mul29(a2, b2);
  }
  return q;
}

template <int V>
__device__ __noinline__ T mul1v(T a, T b) {
  if constexpr (V == 0) return Fr255::mul(a, b);
  else return mul29(a, b);
}

template <int V>
__global__ void k_tput(T* out, const T* in, int iters) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  T x = in[3 * i], y = in[3 * i + 1], z = in[3 * i + 2];
  const T k = in[0];
  for (int it = 0; it < iters; it++) {
    Tri q = mul3v<V>(x, k, y, k, z, k);
    x = q.x; y = q.y; z = q.z;
  }
  out[3 * i] = x; out[3 * i + 1] = y; out[3 * i + 2] = z;
}

template <int V>
__global__ void k_lat(T* out, const T* in, int iters, long long* cyc) {
  T x = in[threadIdx.x];
  const T k = in[0];
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) x = mul1v<V>(x, k);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

static uint64_t s = 88172645463325252ull;
static uint32_t rnd() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (uint32_t)s; }
static T rnd_elem() {
  T a;
  for (int k = 0; k < 8; k++) a.v[k] = rnd();
  a.v[7] &= 0x3fffffffu;
  while (Fr255::geq_p_portable(a)) a = Fr255::sub_p_portable(a);
  return a;
}

static int check() {
  T pm1 = Fr255::modulus(); pm1.v[0] -= 1;
  T edge[4] = {Fr255::zero(), Fr255::one(), pm1, Fr255::r2()};
  int bad = 0;
  for (int it = 0; it < 2000000; it++) {
    T a = it < 16 ? edge[it & 3] : rnd_elem();
    T b = it < 16 ? edge[it >> 2] : rnd_elem();
    T x = Fr255::mul_portable(a, b), y = mul29(a, b);
    if (!Fr255::eq(x, y)) {
      if (bad++ < 5) printf("mismatch at %d\n", it);
    }
  }
  printf("host check: %s (%d mismatches / 2e6)\n", bad ? "FAIL" : "ok", bad);
  return bad != 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && !strcmp(argv[1], "check")) return check();
  if (check()) return 1;
  const int bps = argc > 1 ? atoi(argv[1]) : 2;
  const int iters = argc > 2 ? atoi(argv[2]) : 2000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * bps, n = blocks * threads;
  T* h = (T*)malloc(sizeof(T) * 3 * n);
  for (int i = 0; i < 3 * n; i++) h[i] = rnd_elem();
  T *din, *dout;
  long long* dcyc;
  cudaMalloc(&din, sizeof(T) * 3 * n);
  cudaMalloc(&dout, sizeof(T) * 3 * n);
  cudaMalloc(&dcyc, 8);
  cudaMemcpy(din, h, sizeof(T) * 3 * n, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  T* r[2];
  for (int v = 0; v < 2; v++) {
    auto run = v == 0 ? k_tput<0> : k_tput<1>;
    run<<<blocks, threads>>>(dout, din, 10);
    cudaEventRecord(e0);
    run<<<blocks, threads>>>(dout, din, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    r[v] = (T*)malloc(sizeof(T) * 3 * n);
    cudaMemcpy(r[v], dout, sizeof(T) * 3 * n, cudaMemcpyDeviceToHost);
    printf("%s: %.3e products/s (%d blocks/SM)\n", v == 0 ? "cios32" : "mont29",
           3.0 * n * iters / (ms * 1e-3), bps);
    auto lat = v == 0 ? k_lat<0> : k_lat<1>;
    lat<<<1, 32>>>(dout, din, 1000, dcyc);
    long long cyc;
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    printf("   latency %.0f cycles per dependent product\n", cyc / 1000.0);
  }
  printf("device results %s\n", memcmp(r[0], r[1], sizeof(T) * 3 * n) ? "DIFFER" : "identical");
  cudaError_t e = cudaGetLastError();
  printf("cuda: %s\n", cudaGetErrorString(e));
  return 0;
}
