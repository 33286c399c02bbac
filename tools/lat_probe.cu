// Latency probe for one round of the persistent sumcheck (PROD2 shape):
// per-phase cycle counts of thread 0 when each "round" is separated by an
// idle gap (as when the block waits for the host's challenge).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2508_21393_b200/csrc tools/lat_probe.cu -o lat_probe
#include <cstdio>
#include "common.cuh"
using namespace zkl;
using F = Fr255;
using T = fr_t;

__device__ __forceinline__ long long clk() { return clock64(); }

__global__ void k_probe(T* t0, T* t1, int rounds, int gap_cycles, long long* out, int variant) {
  const int i = threadIdx.x;
  const int half = blockDim.x;
  T r = Fr255::r2();
  long long acc[6] = {0, 0, 0, 0, 0, 0};
  T sink = Fr255::zero();
  for (int j = 0; j < rounds; j++) {
    long long c0 = clk();
    T a0 = ld_cg(t0 + i), b0 = ld_cg(t0 + i + half), a1 = ld_cg(t1 + i), b1 = ld_cg(t1 + i + half);
    T a2 = ld_cg(t0 + i + 2 * half), b2 = ld_cg(t0 + i + 3 * half);
    T a3 = ld_cg(t1 + i + 2 * half), b3 = ld_cg(t1 + i + 3 * half);
    T d0 = F::sub(a2, a0), d1 = F::sub(b2, b0), d2 = F::sub(a3, a1), d3 = F::sub(b3, b1);
    long long c1 = clk();
    if (variant == 0) {
      F::mul4r(r, d0, d1, d2, d3);
    } else if (variant == 1) {
      F::mul2(r, d0, r, d1, d0, d1);
      F::mul2(r, d2, r, d3, d2, d3);
    } else {
      d0 = F::mul(r, d0); d1 = F::mul(r, d1); d2 = F::mul(r, d2); d3 = F::mul(r, d3);
    }
    T f0 = F::add(a0, d0), g0 = F::add(a1, d2);
    T fd = F::sub(F::add(b0, d1), f0), gd = F::sub(F::add(b1, d3), g0);
    long long c2 = clk();
    T p0, p1, pc;
    F::mul3(f0, g0, F::add(f0, fd), F::add(g0, gd), fd, gd, p0, p1, pc);
    long long c3 = clk();
    sink = F::add(sink, F::add(p0, F::add(p1, pc)));
    t0[i] = f0; t1[i] = g0;
    long long c4 = clk();
    __syncthreads();
    long long c5 = clk();
    // idle gap (host round trip)
    while (clk() - c5 < gap_cycles) {
    }
    acc[0] += c1 - c0; acc[1] += c2 - c1; acc[2] += c3 - c2; acc[3] += c4 - c3; acc[4] += c5 - c4;
  }
  if (i == 0) {
    for (int q = 0; q < 5; q++) out[q] = acc[q] / rounds;
    out[7] = sink.v[0];
  }
}

__global__ void k_chain(T* o, int n, long long* out) {
  T a = Fr255::one(), b = Fr255::r2();
  long long c0 = clk();
  for (int i = 0; i < n; i++) a = F::mul(a, b);
  long long c1 = clk();
  T x = a, y = b, z = a;
  for (int i = 0; i < n; i++) F::mul3(x, b, y, b, z, b, x, y, z);
  long long c2 = clk();
  for (int i = 0; i < n; i++) x = F::add(x, y);
  long long c3 = clk();
  o[0] = a; o[1] = x; o[2] = y; o[3] = z;
  out[0] = (c1 - c0) / n; out[1] = (c2 - c1) / n; out[2] = (c3 - c2) / n;
}

int main() {
  T *t0, *t1, *o;
  long long* out;
  const int threads = 256;
  cudaMalloc(&t0, 4 * threads * sizeof(T));
  cudaMalloc(&t1, 4 * threads * sizeof(T));
  cudaMalloc(&o, 256);
  cudaMemset(t0, 1, 4 * threads * sizeof(T));
  cudaMemset(t1, 2, 4 * threads * sizeof(T));
  cudaMallocManaged(&out, 8 * sizeof(long long));
  for (int rep = 0; rep < 2; rep++) {
    k_chain<<<1, 1>>>(o, 200, out);
    cudaDeviceSynchronize();
    printf("warm chains: mul %lld cyc | mul3 %lld cyc | add %lld cyc\n", out[0], out[1], out[2]);
  }
  const char* names[3] = {"mul4r", "2x mul2", "4x mul"};
  for (int v = 0; v < 3; v++)
    for (int gap : {0, 10000, 20000}) {
      k_probe<<<8, threads>>>(t0, t1, 12, gap, out, v);
      cudaDeviceSynchronize();
      printf("fold=%-8s gap=%5d cyc: load %lld | fold %lld | mul3 %lld | store %lld | sync %lld\n",
             names[v], gap, out[0], out[1], out[2], out[3], out[4]);
    }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
