// Pipe rates on this GPU, per thread-op: DFMA, IMAD, IMAD.WIDE.U32, IADD3 with and
// without carry (add.cc/addc chains -> IADD3 / IADD3.X), and DFMA beside IMAD.
// The Montgomery product's pipe bound is built from these.
#include <cstdio>
#include <cstdint>
__global__ void k_dfma(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_imadw(uint64_t* out, int iters) {
  uint64_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  uint32_t b = 0x9e3779b9u + blockIdx.x, c = 12345;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a0) : "r"((uint32_t)a1), "r"(b));
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a1) : "r"((uint32_t)a2), "r"(b));
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a2) : "r"((uint32_t)a3), "r"(b));
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a3) : "r"((uint32_t)a4), "r"(b));
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a4) : "r"((uint32_t)a5), "r"(b));
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a5) : "r"((uint32_t)a6), "r"(b));
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a6) : "r"((uint32_t)a7), "r"(b));
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a7) : "r"((uint32_t)a0), "r"(c));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}
__global__ void k_imad(uint32_t* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  uint32_t b = 0x9e3779b9u + blockIdx.x, c = 12345;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      a0 = a0 * b + c; a1 = a1 * b + c; a2 = a2 * b + c; a3 = a3 * b + c;
      a4 = a4 * b + c; a5 = a5 * b + c; a6 = a6 * b + c; a7 = a7 * b + c;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}
// mixed: the same number of DFMA and IMAD per thread, interleaved (separate pipes?)
__global__ void k_mixed(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  uint32_t i0 = threadIdx.x, i1 = i0 + 1, i2 = i0 + 2, i3 = i0 + 3;
  const double b = 1.0000001, c = 1e-9;
  uint32_t ib = 0x9e3779b9u + blockIdx.x, ic = 12345;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      i0 = i0 * ib + ic; i1 = i1 * ib + ic; i2 = i2 * ib + ic; i3 = i3 * ib + ic;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + (double)(i0 ^ i1 ^ i2 ^ i3);
}

// 3-input adds with carry out / carry in: add.cc + addc.cc chains over 8 words
__global__ void k_addc(uint32_t* out, int iters) {
  uint32_t x[8], w[8];
#pragma unroll
  for (int k = 0; k < 8; k++) { x[k] = threadIdx.x + k; w[k] = blockIdx.x * 7 + k; }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
      asm volatile("add.cc.u32 %0, %0, %8;\n\taddc.cc.u32 %1, %1, %9;\n\taddc.cc.u32 %2, %2, %10;\n\t"
          "addc.cc.u32 %3, %3, %11;\n\taddc.cc.u32 %4, %4, %12;\n\taddc.cc.u32 %5, %5, %13;\n\t"
          "addc.cc.u32 %6, %6, %14;\n\taddc.u32 %7, %7, %15;"
          : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7])
          : "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
      asm volatile("add.cc.u32 %0, %0, %8;\n\taddc.cc.u32 %1, %1, %9;\n\taddc.cc.u32 %2, %2, %10;\n\t"
          "addc.cc.u32 %3, %3, %11;\n\taddc.cc.u32 %4, %4, %12;\n\taddc.cc.u32 %5, %5, %13;\n\t"
          "addc.cc.u32 %6, %6, %14;\n\taddc.u32 %7, %7, %15;"
          : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]), "+r"(w[7])
          : "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7]));
    }
  }
  uint32_t a = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) a ^= x[k] ^ w[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
// plain 3-input adds (IADD3 without carries)
__global__ void k_iadd3(uint32_t* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const uint32_t b = blockIdx.x, c = 12345;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      a0 = a0 + b + c; a1 = a1 ^ b ^ a0; a2 = a2 + b + a1; a3 = a3 ^ c ^ a2;
      a4 = a4 + b + a3; a5 = a5 ^ c ^ a4; a6 = a6 + c + a5; a7 = a7 ^ b ^ a6;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 2000;
  void* buf; cudaMalloc(&buf, (size_t)blocks * threads * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double ops = (double)blocks * threads * iters * 16 * 8;
  for (int rep = 0; rep < 2; rep++) {
    float ms;
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>((double*)buf, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("DFMA       %.2f T/s\n", ops / ms / 1e9);
    cudaEventRecord(e0); k_imadw<<<blocks, threads>>>((uint64_t*)buf, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("IMAD.WIDE  %.2f T/s\n", ops / ms / 1e9);
    cudaEventRecord(e0); k_imad<<<blocks, threads>>>((uint32_t*)buf, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("IMAD       %.2f T/s\n", ops / ms / 1e9);
    cudaEventRecord(e0); k_mixed<<<blocks, threads>>>((double*)buf, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("mixed DFMA+IMAD %.2f T/s (each)\n", ops / 2 / ms / 1e9);
    cudaEventRecord(e0); k_addc<<<blocks, threads>>>((uint32_t*)buf, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("add.cc/addc chain words %.2f T/s\n", (double)blocks * threads * iters * 4 * 16 / ms / 1e9);
    cudaEventRecord(e0); k_iadd3<<<blocks, threads>>>((uint32_t*)buf, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("IADD3/LOP3 %.2f T/s\n", ops / ms / 1e9);
  }
  return 0;
}
