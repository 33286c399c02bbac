#include <cstdio>
#include <cstdint>
#include <cstring>
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
struct alignas(128) Box { volatile uint64_t ev[72]; volatile uint64_t ch[8]; };
// MODE 0: lanes 0..7 scalar 8B loads; 1: lanes 0..3 v2 loads; 2: lane 0 scalar 1 word; 3: lanes 0..2 v2 (3 x 16B)
template <int MODE>
__global__ void k(Box* b, int iters, uint64_t* out) {
  const int lane = threadIdx.x;
  uint64_t t0 = gtime();
  for (int i = 1; i <= iters; i++) {
    if (lane == 0) b->ev[0] = (uint64_t)i << 32;
    bool ok = false;
    for (uint64_t ts = gtime(); !ok && gtime() - ts < 200000000ull;) {
      uint64_t a = (uint64_t)i << 32, c = a;
      if (MODE == 0 && lane < 8) a = b->ch[lane];
      if (MODE == 2 && lane < 1) a = b->ch[0];
      if ((MODE == 1 && lane < 4) || (MODE == 3 && lane < 3))
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(c) : "l"(b->ch + 2 * lane) : "memory");
      ok = __all_sync(0xffffffff, (a >> 32) == (uint64_t)i && (c >> 32) == (uint64_t)i);
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
  const char* names[] = {"8 lanes x 8B", "4 lanes x 16B", "1 lane x 8B", "3 lanes x 16B"};
  for (int mode = 0; mode < 4; mode++) {
    memset((void*)h, 0, sizeof(Box));
    if (mode == 0) k<0><<<1, 32>>>(d, iters, out);
    if (mode == 1) k<1><<<1, 32>>>(d, iters, out);
    if (mode == 2) k<2><<<1, 32>>>(d, iters, out);
    if (mode == 3) k<3><<<1, 32>>>(d, iters, out);
    bool dead = false;
    for (int i = 1; i <= iters && !dead; i++) {
      for (long sp = 0; (h->ev[0] >> 32) != (uint64_t)i; sp++) if (sp > 400000000L) { dead = true; break; }
      for (int w = 0; w < 8; w++) h->ch[w] = (uint64_t)i << 32 | w;
    }
    cudaDeviceSynchronize();
    printf("%-14s: round trip %.0f ns %s\n", names[mode], (double)out[0], dead ? "(STUCK)" : "");
    fflush(stdout);
  }
}
