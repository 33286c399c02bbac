#include <cstdio>
#include <cstdint>
#include <cstring>
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
struct alignas(128) Box { volatile uint64_t ev[72]; volatile uint64_t ch[8]; };
template <int MODE>
__device__ __forceinline__ void ld2(const volatile uint64_t* p, uint64_t& a, uint64_t& b) {
  if (MODE == 0) asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  if (MODE == 1) asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  if (MODE == 2) asm volatile("ld.global.cv.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
template <int MODE>
__global__ void k(Box* b, int iters, int lanes_read, uint64_t* out) {
  const int lane = threadIdx.x;
  uint64_t t0 = gtime();
  for (int i = 1; i <= iters; i++) {
    if (lane == 0) b->ev[0] = (uint64_t)i << 32;
    if (lanes_read == 1) {
      if (lane == 0) for (uint64_t ts = gtime(); gtime() - ts < 200000000ull;) {
        bool ok = true;
        for (int w = 0; w < 8; w += 2) { uint64_t a, c; ld2<MODE>(b->ch + w, a, c); ok &= (a >> 32) == (uint64_t)i && (c >> 32) == (uint64_t)i; }
        if (ok) break;
      }
    } else {
      bool ok = false;
      for (uint64_t ts = gtime(); !ok && gtime() - ts < 200000000ull;) {
        uint64_t a = (uint64_t)i << 32, c = a;
        if (lane < 4) ld2<MODE>(b->ch + 2 * lane, a, c);
        ok = __all_sync(0xffffffff, (a >> 32) == (uint64_t)i && (c >> 32) == (uint64_t)i);
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
  const char* names[] = {"volatile", "relaxed.sys", "cv"};
  for (int mode = 0; mode < 3; mode++) for (int lr : {1, 4}) {
    memset((void*)h, 0, sizeof(Box));
    if (mode == 0) k<0><<<1, 32>>>(d, iters, lr, out);
    if (mode == 1) k<1><<<1, 32>>>(d, iters, lr, out);
    if (mode == 2) k<2><<<1, 32>>>(d, iters, lr, out);
    bool dead = false;
    for (int i = 1; i <= iters && !dead; i++) {
      for (long sp = 0; (h->ev[0] >> 32) != (uint64_t)i; sp++) if (sp > 400000000L) { dead = true; break; }
      for (int w = 0; w < 8; w++) h->ch[w] = (uint64_t)i << 32 | w;
    }
    cudaDeviceSynchronize();
    printf("%-12s %s: round trip %.0f ns %s\n", names[mode], lr == 1 ? "1 lane x 4 loads" : "4 lanes x 1 load", (double)out[0], dead ? "(STUCK)" : "");
    fflush(stdout);
  }
}
