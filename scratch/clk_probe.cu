#include <cstdio>
#include <cstdint>
#include <ctime>
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(volatile uint64_t* b, uint64_t* out, int iters) {
  for (int i = 1; i <= iters; i++) {
    uint64_t t = gtime();
    b[0] = t;          // payload: device time
    b[1] = i;
    while (b[8] != (uint64_t)i) {}
    out[i] = gtime();  // device time when reply seen
  }
}
static uint64_t now_ns() { timespec ts; clock_gettime(CLOCK_REALTIME, &ts); return ts.tv_sec * 1000000000ull + ts.tv_nsec; }
int main() {
  volatile uint64_t* h; cudaHostAlloc((void**)&h, 4096, cudaHostAllocMapped);
  for (int i = 0; i < 64; i++) h[i] = 0;
  uint64_t* d; cudaHostGetDevicePointer((void**)&d, (void*)h, 0);
  uint64_t* out; cudaMallocManaged(&out, 8 * 1001);
  const int iters = 1000;
  static uint64_t seen[1001], dev_sent[1001], host_reply[1001];
  k<<<1, 1>>>(d, out, iters);
  for (int i = 1; i <= iters; i++) {
    while (h[1] != (uint64_t)i) {}
    seen[i] = now_ns(); dev_sent[i] = h[0];
    host_reply[i] = now_ns();
    h[8] = i;
  }
  cudaDeviceSynchronize();
  double a = 0, b = 0, c = 0;
  for (int i = 100; i <= iters; i++) { a += (double)(int64_t)(seen[i] - dev_sent[i]); b += (double)(int64_t)(out[i] - host_reply[i]); c += (double)(out[i] - dev_sent[i]); }
  int n = iters - 99;
  printf("dev->host %.0f ns | host->dev %.0f ns | round trip %.0f ns (clock offset cancels in the sum)\n", a / n, b / n, c / n);
  return 0;
}
