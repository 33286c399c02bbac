#include <cstdio>
#include <cstdint>
#include <cstring>
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
struct alignas(128) Box { volatile uint64_t ev[72]; volatile uint64_t ch[8]; };
__device__ __forceinline__ void st2(volatile uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory"); }
__device__ __forceinline__ void ld2(const volatile uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory"); }
__global__ void k(Box* b, int iters, int nwrite, int nread, uint64_t* out) {
  const int lane = threadIdx.x;
  uint64_t t0 = gtime();
  for (int i = 1; i <= iters; i++) {
    for (int idx = 2 * lane; idx < nwrite; idx += 64) st2(b->ev + idx, (uint64_t)i << 32, (uint64_t)i << 32);
    if (nwrite == 1 && lane == 0) b->ev[0] = (uint64_t)i << 32;
    if (lane == 0) {
      while (true) {
        bool ok = true;
        for (int w = 0; w < nread; w += 2) { uint64_t a, c; ld2(b->ch + w, a, c); ok &= (a >> 32) == (uint64_t)i; }
        if (ok) break;
      }
    }
    __syncwarp();
  }
  if (lane == 0) out[0] = (gtime() - t0) / iters;
}
int main() {
  Box* h; cudaHostAlloc((void**)&h, sizeof(Box), cudaHostAllocMapped);
  Box* d; cudaHostGetDevicePointer((void**)&d, h, 0);
  uint64_t* out; cudaMallocManaged(&out, 64);
  const int iters = 2000;
  int cfgs[][2] = {{1, 2}, {1, 8}, {28, 2}, {28, 8}, {54, 8}};
  for (auto& c : cfgs) {
    memset((void*)h, 0, sizeof(Box));
    k<<<1, 32>>>(d, iters, c[0], c[1], out);
    for (int i = 1; i <= iters; i++) {
      const int nw = c[0];
      while (true) { bool ok = true; for (int w = 0; w < nw; w++) ok &= (h->ev[w] >> 32) == (uint64_t)i; if (ok) break; }
      for (int w = 0; w < 8; w++) h->ch[w] = (uint64_t)i << 32 | w;
    }
    cudaDeviceSynchronize();
    printf("write %2d words, read %d words: round trip %.0f ns\n", c[0], c[1], (double)out[0]);
  }
}
