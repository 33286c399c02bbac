// Device <-> host mailbox round-trip probe (mapped pinned memory).
//   device: store tagged word -> poll host reply;  host: spin, reply.
// Variants: 1 polling lane, and K lanes polling with staggered start.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/pcie_probe.cu -o pcie_probe
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <thread>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct alignas(128) Box {
  volatile uint64_t dev[16];
  volatile uint64_t host[16];
};

__global__ void k_ping(Box* b, int iters, int lanes, int stagger_ns, uint64_t* out) {
  __shared__ volatile int got;
  const int lane = threadIdx.x;
  uint64_t t0 = gtime();
  for (int i = 1; i <= iters; i++) {
    if (lane == 0) {
      got = 0;
      b->dev[0] = (uint64_t)i;
    }
    __syncwarp();
    if (lane < lanes) {
      // staggered start
      const uint64_t ts = gtime();
      while (gtime() - ts < (uint64_t)(lane * stagger_ns)) {
      }
      while (!got) {
        uint64_t v = b->host[0];
        if (v == (uint64_t)i) {
          got = 1;
          break;
        }
      }
    }
    __syncwarp();
  }
  uint64_t t1 = gtime();
  if (lane == 0) out[0] = (t1 - t0) / iters;
}

int main() {
  Box* h;
  cudaHostAlloc((void**)&h, sizeof(Box), cudaHostAllocMapped);
  memset((void*)h, 0, sizeof(Box));
  Box* d;
  cudaHostGetDevicePointer((void**)&d, h, 0);
  uint64_t* out;
  cudaMallocManaged(&out, 64);
  const int iters = 3000;
  for (int lanes : {1, 2, 4, 8})
    for (int stagger : {0, 150, 300}) {
      if (lanes == 1 && stagger) continue;
      memset((void*)h, 0, sizeof(Box));
      k_ping<<<1, 32>>>(d, iters, lanes, stagger, out);
      for (int i = 1; i <= iters; i++) {
        while (h->dev[0] != (uint64_t)i) {
        }
        h->host[0] = (uint64_t)i;
      }
      cudaDeviceSynchronize();
      printf("lanes=%d stagger=%dns: round trip %.0f ns\n", lanes, stagger, (double)out[0]);
    }
  return 0;
}
