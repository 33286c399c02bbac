// mma.sync.m16n8k32 u8 issue rate on this GPU (the legacy tensor-core path the
// byte-sliced matvec / GEMM kernels use): MACs per cycle per SM.
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ void mma_u8(uint32_t (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__global__ void k(uint32_t* out, int iters) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3, threadIdx.x * 5, threadIdx.x * 7};
  uint32_t acc[8][4] = {};
  uint32_t b0 = blockIdx.x, b1 = blockIdx.x * 11;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) mma_u8(acc[j], a, b0 + j, b1);
  }
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s ^= acc[j][0] ^ acc[j][1] ^ acc[j][2] ^ acc[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* o;
  cudaMalloc(&o, 1 << 24);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int wpb : {4, 8, 16}) {
    const int blocks = sms * 2, threads = 32 * wpb, iters = 20000;
    k<<<blocks, threads>>>(o, 10);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = (double)blocks * (threads / 32) * iters * 8;
    printf("warps/SM %2d: %.3e mma/s = %.1f TOPS int8 (%.0f MACs/cycle/SM at 1.965 GHz)\n", 2 * wpb,
           mmas / (ms * 1e-3), mmas * 4096 * 2 / (ms * 1e-3) / 1e12,
           mmas * 4096 / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
