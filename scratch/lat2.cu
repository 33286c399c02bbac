#include <cstdio>
#include "../paper_2508_21393_b200/csrc/common.cuh"
using namespace zkl;
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(fr_t* out, long long* res) {
  fr_t a = Fr255::one(), b = Fr255::r2();
  __syncwarp();
  long long c0 = clock64(); unsigned long long t0 = gt();
  for (int i = 0; i < 2000; i++) a = Fr255::mul(a, b);
  long long c1 = clock64(); unsigned long long t1 = gt();
  fr_t s = warp_sum<Fr255>(a);
  long long c2 = clock64(); unsigned long long t2 = gt();
  for (int i = 0; i < 200; i++) s = warp_sum<Fr255>(s);
  long long c3 = clock64(); unsigned long long t3 = gt();
  fr_t x = a;
  for (int i = 0; i < 2000; i++) x = Fr255::add(x, b);
  long long c4 = clock64(); unsigned long long t4 = gt();
  if (threadIdx.x == 0) {
    out[0] = s; out[1] = x;
    res[0] = c1 - c0; res[1] = t1 - t0; res[2] = c3 - c2; res[3] = t3 - t2; res[4] = c4 - c3; res[5] = t4 - t3;
  }
}
int main() {
  fr_t* o; long long* r; cudaMalloc(&o, 128); cudaMallocManaged(&r, 64);
  for (int rep = 0; rep < 3; rep++) {
    k<<<1, 32>>>(o, r); cudaDeviceSynchronize();
    printf("mul: %.0f cyc %.1f ns (%.0f MHz) | warp_sum: %.0f cyc %.1f ns | add: %.1f cyc %.2f ns\n",
           r[0] / 2000.0, r[1] / 2000.0, r[0] * 1000.0 / r[1], r[2] / 200.0, r[3] / 200.0, r[4] / 2000.0, r[5] / 2000.0);
  }
  return 0;
}
