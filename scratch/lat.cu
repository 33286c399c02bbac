// Latency microbenchmarks: mont-mul chain, block_sum, mailbox ping-pong.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>

#include "../paper_2508_21393_b200/csrc/common.cuh"

using namespace zkl;

__global__ void k_mul_chain(fr_t* out, int iters, long long* cyc) {
  fr_t a = Fr255::one(), b = Fr255::r2();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) a = Fr255::mul(a, b);
  long long t1 = clock64();
  out[0] = a;
  cyc[0] = t1 - t0;
}

__global__ void k_blocksum(fr_t* out, int iters, long long* cyc) {
  __shared__ fr_t sm[32];
  fr_t v[4] = {Fr255::one(), Fr255::one(), Fr255::one(), Fr255::one()};
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) block_sum<Fr255, 4>(v, sm);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = v[0]; cyc[0] = t1 - t0; }
}

struct alignas(64) Box {
  volatile unsigned dev_seq;
  volatile unsigned host_seq;
};

__global__ void k_pingpong(Box* b, int iters, unsigned long long* ns) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; i++) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(&b->dev_seq), "r"(i) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(&b->host_seq) : "memory");
    } while (v != (unsigned)i);
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  *ns = t1 - t0;
}

int main() {
  fr_t* out;
  long long* cyc;
  cudaMalloc(&out, 64);
  cudaMallocManaged(&cyc, 64);
  k_mul_chain<<<1, 1>>>(out, 1000, cyc);
  cudaDeviceSynchronize();
  k_mul_chain<<<1, 1>>>(out, 1000, cyc);
  cudaDeviceSynchronize();
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("mont mul chain: %.1f cycles/mul\n", cyc[0] / 1000.0);
  k_blocksum<<<1, 256>>>(out, 100, cyc);
  cudaDeviceSynchronize();
  printf("block_sum<4> (256 thr): %.1f cycles\n", cyc[0] / 100.0);

  Box* h;
  cudaHostAlloc((void**)&h, sizeof(Box), cudaHostAllocMapped);
  h->dev_seq = 0;
  h->host_seq = 0;
  Box* d;
  cudaHostGetDevicePointer((void**)&d, h, 0);
  unsigned long long* ns;
  cudaMallocManaged(&ns, 8);
  const int iters = 2000;
  auto t0 = std::chrono::steady_clock::now();
  k_pingpong<<<1, 1>>>(d, iters, ns);
  for (int i = 1; i <= iters; i++) {
    while (h->dev_seq != (unsigned)i) {
    }
    std::atomic_thread_fence(std::memory_order_seq_cst);
    h->host_seq = i;
  }
  cudaDeviceSynchronize();
  auto t1 = std::chrono::steady_clock::now();
  printf("mailbox ping-pong: device %.2f us/round, host %.2f us/round\n", *ns / 1000.0 / iters,
         std::chrono::duration<double, std::micro>(t1 - t0).count() / iters);
  // launch + sync latency
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 1000; i++) {
    k_mul_chain<<<1, 1>>>(out, 1, cyc);
    cudaStreamSynchronize(0);
  }
  t1 = std::chrono::steady_clock::now();
  printf("launch+sync: %.2f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 1000);
  return 0;
}
