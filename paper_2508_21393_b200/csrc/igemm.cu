// Exact int16 x int16 -> int64 GEMM on the tensor cores, for the LoRA-block
// witness (the wide products every zkMat / rescale gadget takes as its claim,
// model.py:479-487 computes them with a Python triple loop).
//
// Each int16 entry is split into a signed high byte and an unsigned low byte,
// a = 256 ah + al, so
//   A B = 2^16 (Ah Bh) + 2^8 (Ah Bl + Al Bh) + (Al Bl),
// four byte GEMMs on mma.sync.m16n8k32 (s8 / u8 operands, s32 accumulators).
// The two cross terms share one accumulator.  With K <= 2^14 per chunk every
// int32 sum is exact: |Ah Bh| < 2^14 K, |Ah Bl + Al Bh| < 2^16 K, Al Bl < 2^16 K;
// longer contractions flush the chunk sums into int64 every 2^14 columns.
//
// CTA tile 128 x 64 outputs, 8 warps as 4 (M) x 2 (N), each warp 32 x 32
// (2 m16 x 4 n8 mma tiles); K steps of 32 staged in shared memory (A
// row-major, B transposed so a B fragment is two 32-bit loads); out-of-range
// rows / columns / k are zero-filled, so any M, N, K works.
#include <cstdint>

#include "common.cuh"
#include "ops.cuh"

namespace zkl {

namespace {

constexpr int kTM = 128, kTN = 64, kTK = 32;
constexpr int kKChunk = 1 << 14;
constexpr int kAPitch = kTK + 8;  // int16 per smem row (16-byte skew)
constexpr int kBPitch = kTK + 8;

ZKL_D void mma_s8s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
ZKL_D void mma_s8u8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
ZKL_D void mma_u8s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
ZKL_D void mma_u8u8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// 4 consecutive int16 (two 32-bit words) -> (high bytes, low bytes), k order kept
ZKL_D void split4(uint32_t w0, uint32_t w1, uint32_t& hi, uint32_t& lo) {
  hi = __byte_perm(w0, w1, 0x7531);
  lo = __byte_perm(w0, w1, 0x6420);
}

__global__ void __launch_bounds__(256)
    k_igemm16(const int16_t* __restrict__ A, const int16_t* __restrict__ B,
              int64_t* __restrict__ C, int M, int K, int N) {
  __shared__ __align__(16) int16_t sa[kTM * kAPitch];
  __shared__ __align__(16) int16_t sb[kTN * kBPitch];  // transposed: [n][k]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;  // warp tile origin (wm * 32, wn * 32)
  const int m0 = blockIdx.y * kTM, n0 = blockIdx.x * kTN;
  long long tot[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int q = 0; q < 4; q++) tot[i][j][q] = 0;
  for (int kc = 0; kc < K; kc += kKChunk) {
    const int kend = kc + kKChunk < K ? kc + kKChunk : K;
    int hh[2][4][4], mx[2][4][4], ll[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int q = 0; q < 4; q++) hh[i][j][q] = mx[i][j][q] = ll[i][j][q] = 0;
    for (int k0 = kc; k0 < kend; k0 += kTK) {
      // stage A (128 x 32): each thread two rows' 8-entry runs
#pragma unroll
      for (int rep = 0; rep < 2; rep++) {
        const int e = tid + rep * 256;  // 512 runs of 8
        const int r = e >> 2, c8 = (e & 3) * 8;
        const int gr = m0 + r, gc = k0 + c8;
        int16_t v[8];
        if (gr < M && gc + 8 <= kend && ((reinterpret_cast<uintptr_t>(A + (size_t)gr * K + gc) & 15) == 0)) {
          *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(A + (size_t)gr * K + gc);
        } else {
#pragma unroll
          for (int t = 0; t < 8; t++)
            v[t] = (gr < M && gc + t < kend) ? A[(size_t)gr * K + gc + t] : (int16_t)0;
        }
        *reinterpret_cast<uint4*>(sa + r * kAPitch + c8) = *reinterpret_cast<uint4*>(v);
      }
      // stage B (32 x 64) transposed into sb[n][k]
      {
        const int r = tid >> 3, c8 = (tid & 7) * 8;  // 256 runs of 8 along n
        const int gr = k0 + r, gc = n0 + c8;
        int16_t v[8];
        if (gr < kend && gc + 8 <= N && ((reinterpret_cast<uintptr_t>(B + (size_t)gr * N + gc) & 15) == 0)) {
          *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(B + (size_t)gr * N + gc);
        } else {
#pragma unroll
          for (int t = 0; t < 8; t++)
            v[t] = (gr < kend && gc + t < N) ? B[(size_t)gr * N + gc + t] : (int16_t)0;
        }
#pragma unroll
        for (int t = 0; t < 8; t++) sb[(c8 + t) * kBPitch + r] = v[t];
      }
      __syncthreads();
      // fragments: A rows wm*32 + i*16 + {g, g+8}, k slots 4 tig.. and 16 + 4 tig..
      uint32_t ahi[2][4], alo[2][4];
#pragma unroll
      for (int i = 0; i < 2; i++) {
        const int rb = wm * 32 + i * 16;
#pragma unroll
        for (int h = 0; h < 2; h++) {      // k half: 0 -> slots 0..15, 1 -> 16..31
#pragma unroll
          for (int rr = 0; rr < 2; rr++) {  // row g / g + 8
            const int16_t* p = sa + (rb + g + 8 * rr) * kAPitch + 16 * h + 4 * tig;
            const uint2 w = *reinterpret_cast<const uint2*>(p);
            split4(w.x, w.y, ahi[i][2 * h + rr], alo[i][2 * h + rr]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int cb = wn * 32 + j * 8 + g;  // this thread's B column
        const int16_t* p = sb + cb * kBPitch + 4 * tig;
        const uint2 w0 = *reinterpret_cast<const uint2*>(p);
        const uint2 w1 = *reinterpret_cast<const uint2*>(p + 16);
        uint32_t bh0, bl0, bh1, bl1;
        split4(w0.x, w0.y, bh0, bl0);
        split4(w1.x, w1.y, bh1, bl1);
#pragma unroll
        for (int i = 0; i < 2; i++) {
          mma_s8s8(hh[i][j], ahi[i], bh0, bh1);
          mma_s8u8(mx[i][j], ahi[i], bl0, bl1);
          mma_u8s8(mx[i][j], alo[i], bh0, bh1);
          mma_u8u8(ll[i][j], alo[i], bl0, bl1);
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int q = 0; q < 4; q++)
          tot[i][j][q] += ((long long)hh[i][j][q] << 16) + ((long long)mx[i][j][q] << 8) +
                          (long long)(unsigned)ll[i][j][q];
  }
  // C fragment: c0, c1 -> row g, cols 2 tig, 2 tig + 1; c2, c3 -> row g + 8
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int r = m0 + wm * 32 + i * 16 + g + 8 * (q >> 1);
        const int c = n0 + wn * 32 + j * 8 + 2 * tig + (q & 1);
        if (r < M && c < N) C[(size_t)r * N + c] = tot[i][j][q];
      }
}

}  // namespace

int op_igemm16(const int16_t* A, const int16_t* B, int64_t* C, int M, int K, int N,
               cudaStream_t s) {
  if (M <= 0 || N <= 0 || K < 0) {
    set_error("igemm16: bad shape %d x %d x %d", M, K, N);
    return kErrArg;
  }
  if (K == 0) {
    ZKL_CUDA(cudaMemsetAsync(C, 0, (size_t)M * N * 8, s));
    return kOk;
  }
  dim3 grid((N + kTN - 1) / kTN, (M + kTM - 1) / kTM);
  if (grid.y > 65535) {
    set_error("igemm16: M = %d too large", M);
    return kErrArg;
  }
  k_igemm16<<<grid, 256, 0, s>>>(A, B, C, M, K, N);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

}  // namespace zkl
