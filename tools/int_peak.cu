// Integer / FP64 pipe throughput on this GPU (the IMAD roofline denominator
// for the field-arithmetic kernels).  Each thread runs 8 independent chains
// of the instruction under test; the grid fills every SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/int_peak.cu -o int_peak
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 4096;

__global__ void k_imad(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; i++) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imad_wide(uint64_t* out, uint32_t a) {
  uint64_t x[8];
  uint32_t m[8];
  for (int i = 0; i < 8; i++) { x[i] = threadIdx.x + i; m[i] = threadIdx.x * 7 + i; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(x[i]) : "r"(m[i]), "r"(a));
  }
  uint64_t s = 0;
  for (int i = 0; i < 8; i++) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// IMAD.WIDE.U32 with a zero addend (mul.wide.u32): chains through the low word
__global__ void k_mul_wide(uint64_t* out, uint32_t a) {
  uint64_t x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("{ .reg .u32 t; cvt.u32.u64 t, %0; mul.wide.u32 %0, t, %1; }" : "+l"(x[i]) : "r"(a));
  }
  uint64_t s = 0;
  for (int i = 0; i < 8; i++) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imad_hi(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; i++) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_iadd3(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; i++) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[i]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; i++) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256;
  void* buf;
  cudaMalloc(&buf, (size_t)blocks * threads * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double ops = (double)blocks * threads * ITERS * 8;
  auto run = [&](const char* name, auto launch, double per) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double rate = ops * per * 5 / (ms * 1e-3);
    printf("%-14s %8.2f T thread-ops/s  = %6.1f per SM per clk at %d MHz boost\n", name,
           rate / 1e12, rate / sms / (clk * 1e3), clk / 1000);
  };
  run("IMAD (lo)", [&] { k_imad<<<blocks, threads>>>((uint32_t*)buf, 3, 5); }, 1);
  run("mad.wide acc", [&] { k_imad_wide<<<blocks, threads>>>((uint64_t*)buf, 3); }, 1);
  run("mul.wide(RZ)", [&] { k_mul_wide<<<blocks, threads>>>((uint64_t*)buf, 3); }, 1);
  run("IMAD.HI", [&] { k_imad_hi<<<blocks, threads>>>((uint32_t*)buf, 3, 5); }, 1);
  run("IADD3 (x2)", [&] { k_iadd3<<<blocks, threads>>>((uint32_t*)buf, 3, 5); }, 2);
  run("DFMA", [&] { k_dfma<<<blocks, threads>>>((double*)buf, 1.0000001, 0.5); }, 1);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
