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
// (2 m16 x 4 n8 mma tiles); K steps of 64 staged in shared memory (A
// row-major, B transposed so a B fragment is two 32-bit loads), two stages:
// step s+1 is loaded into registers while step s feeds the MMAs.  Out-of-range
// rows / columns / k are zero-filled, so any M, N, K works.
#include <cstdint>

#include "common.cuh"
#include "ops.cuh"

namespace zkl {

namespace {

constexpr int kTM = 128, kTN = 64, kTK = 64;
constexpr int kKChunk = 1 << 14;
constexpr int kPitch = kTK + 8;  // int16 per smem row (16-byte skew)
constexpr int kStage = (kTM + kTN) * kPitch;  // int16 per pipeline stage

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

// one K step's global tile in registers: A 128 x 64 (4 runs of 8 per thread),
// B 64 x 64 (2 runs of 8 along n per thread); zero outside the matrices
struct Regs {
  uint4 a[4];
  uint4 b[2];
};

ZKL_D uint4 load8(const int16_t* base, bool full, int row_ok, int avail) {
  if (full) return *reinterpret_cast<const uint4*>(base);
  int16_t v[8];
#pragma unroll
  for (int t = 0; t < 8; t++) v[t] = (row_ok && t < avail) ? base[t] : (int16_t)0;
  return *reinterpret_cast<uint4*>(v);
}

ZKL_D void fetch(Regs& R, const int16_t* A, const int16_t* B, int M, int K, int N, int m0, int n0,
                 int k0, int kend, int tid, bool a_al, bool b_al) {
#pragma unroll
  for (int rep = 0; rep < 4; rep++) {
    const int e = tid + rep * 256;  // 1024 runs of 8: row e / 8, k 8 (e % 8)
    const int r = e >> 3, c8 = (e & 7) * 8;
    const int gr = m0 + r, gc = k0 + c8;
    const int avail = kend - gc;
    R.a[rep] = load8(A + (size_t)(gr < M ? gr : 0) * K + (gc < kend ? gc : 0),
                     a_al && gr < M && avail >= 8, gr < M, avail);
  }
#pragma unroll
  for (int rep = 0; rep < 2; rep++) {
    const int e = tid + rep * 256;  // 512 runs of 8 along n: k row e / 8
    const int r = e >> 3, c8 = (e & 7) * 8;
    const int gr = k0 + r, gc = n0 + c8;
    const int avail = N - gc;
    R.b[rep] = load8(B + (size_t)(gr < kend ? gr : 0) * N + (gc < N ? gc : 0),
                     b_al && gr < kend && avail >= 8, gr < kend, avail);
  }
}

ZKL_D void stash(const Regs& R, int16_t* st, int tid) {
  int16_t* sa = st;
  int16_t* sb = st + kTM * kPitch;  // transposed: [n][k]
#pragma unroll
  for (int rep = 0; rep < 4; rep++) {
    const int e = tid + rep * 256;
    *reinterpret_cast<uint4*>(sa + (e >> 3) * kPitch + (e & 7) * 8) = R.a[rep];
  }
#pragma unroll
  for (int rep = 0; rep < 2; rep++) {
    const int e = tid + rep * 256;
    const int r = e >> 3, c8 = (e & 7) * 8;
    const int16_t* v = reinterpret_cast<const int16_t*>(&R.b[rep]);
#pragma unroll
    for (int t = 0; t < 8; t++) sb[(c8 + t) * kPitch + r] = v[t];
  }
}

__global__ void __launch_bounds__(256)
    k_igemm16(const int16_t* __restrict__ A, const int16_t* __restrict__ B,
              int64_t* __restrict__ C, int M, int K, int N, int kslice) {
  extern __shared__ __align__(16) int16_t smem[];  // 2 stages
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;  // warp tile origin (wm * 32, wn * 32)
  const int m0 = blockIdx.y * kTM, n0 = blockIdx.x * kTN;
  const bool a_al = (K & 7) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  const bool b_al = (N & 7) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
  long long tot[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int q = 0; q < 4; q++) tot[i][j][q] = 0;
  // split-K (skinny products): blockIdx.z takes K columns [kb, ke) and adds
  // its partial sums into the zeroed output
  const int kb = blockIdx.z * kslice;
  const int ke = kb + kslice < K ? kb + kslice : K;
  for (int kc = kb; kc < ke; kc += kKChunk) {
    const int kend = kc + kKChunk < ke ? kc + kKChunk : ke;
    int hh[2][4][4], mx[2][4][4], ll[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int q = 0; q < 4; q++) hh[i][j][q] = mx[i][j][q] = ll[i][j][q] = 0;
    // software pipeline: the next step's tile is in registers while this
    // step's (in shared memory) feeds the MMAs; two shared stages
    Regs R;
    fetch(R, A, B, M, K, N, m0, n0, kc, kend, tid, a_al, b_al);
    stash(R, smem, tid);
    __syncthreads();
    int stage = 0;
    for (int k0 = kc; k0 < kend; k0 += kTK) {
      const bool more = k0 + kTK < kend;
      if (more) fetch(R, A, B, M, K, N, m0, n0, k0 + kTK, kend, tid, a_al, b_al);
      const int16_t* sa = smem + stage * kStage;
      const int16_t* sb = sa + kTM * kPitch;
#pragma unroll
      for (int ks = 0; ks < kTK; ks += 32) {
        uint32_t ahi[2][4], alo[2][4];
#pragma unroll
        for (int i = 0; i < 2; i++) {
          const int rb = wm * 32 + i * 16;
#pragma unroll
          for (int h = 0; h < 2; h++)
#pragma unroll
            for (int rr = 0; rr < 2; rr++) {
              const int16_t* p = sa + (rb + g + 8 * rr) * kPitch + ks + 16 * h + 4 * tig;
              const uint2 w = *reinterpret_cast<const uint2*>(p);
              split4(w.x, w.y, ahi[i][2 * h + rr], alo[i][2 * h + rr]);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int16_t* p = sb + (wn * 32 + j * 8 + g) * kPitch + ks + 4 * tig;
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
      }
      if (more) {
        stage ^= 1;
        stash(R, smem + stage * kStage, tid);  // the other stage: nobody reads it now
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
      for (int q = 0; q < 4; q += 2) {
        const int r = m0 + wm * 32 + i * 16 + g + 8 * (q >> 1);
        const int c = n0 + wn * 32 + j * 8 + 2 * tig;
        if (gridDim.z > 1) {  // two's complement partial sums add exactly mod 2^64
          unsigned long long* d = reinterpret_cast<unsigned long long*>(C + (size_t)r * N + c);
          if (r < M && c < N) atomicAdd(d, (unsigned long long)tot[i][j][q]);
          if (r < M && c + 1 < N) atomicAdd(d + 1, (unsigned long long)tot[i][j][q + 1]);
        } else if (r < M && c + 1 < N && ((N & 1) == 0)) {
          *reinterpret_cast<longlong2*>(C + (size_t)r * N + c) =
              make_longlong2(tot[i][j][q], tot[i][j][q + 1]);
        } else {
          if (r < M && c < N) C[(size_t)r * N + c] = tot[i][j][q];
          if (r < M && c + 1 < N) C[(size_t)r * N + c + 1] = tot[i][j][q + 1];
        }
      }
}

// int16 -> int8 planes for a library int8 GEMM: hi = a >> 8 (signed), lo =
// (a & 255) - 128 (signed), so a = 256 hi + lo + 128; 8 entries per thread
__global__ void k_split16(const int16_t* __restrict__ src, uint64_t n, int8_t* __restrict__ hi,
                          int8_t* __restrict__ lo) {
  const uint64_t i8 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 8;
  if (i8 + 8 <= n && (((uintptr_t)src | (uintptr_t)hi | (uintptr_t)lo) & 15) == 0) {
    const uint4 v = *reinterpret_cast<const uint4*>(src + i8);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t h[2], l[2];
#pragma unroll
    for (int q = 0; q < 2; q++) {
      h[q] = __byte_perm(w[2 * q], w[2 * q + 1], 0x7531);
      l[q] = __byte_perm(w[2 * q], w[2 * q + 1], 0x6420) ^ 0x80808080u;  // - 128
    }
    *reinterpret_cast<uint2*>(hi + i8) = make_uint2(h[0], h[1]);
    *reinterpret_cast<uint2*>(lo + i8) = make_uint2(l[0], l[1]);
  } else {
    for (uint64_t i = i8; i < n && i < i8 + 8; i++) {
      const int v = src[i];
      hi[i] = (int8_t)(v >> 8);
      lo[i] = (int8_t)((v & 255) - 128);
    }
  }
}

// C = 65536 HH + 256 (HL + LH) + LL + 128 (rowA_i + colB_j) - 16384 K: the
// exact int64 product from the four int8 plane products (int32) and the
// operands' row / column sums
__global__ void k_igemm_combine(const int32_t* __restrict__ hh, const int32_t* __restrict__ hl,
                                const int32_t* __restrict__ lh, const int32_t* __restrict__ ll,
                                const int64_t* __restrict__ rowA, const int64_t* __restrict__ colB,
                                int64_t K, int64_t* __restrict__ C, int M, int N) {
  const uint64_t n = (uint64_t)M * N;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / N, c = i % N;
    C[i] = 65536ll * hh[i] + 256ll * ((int64_t)hl[i] + lh[i]) + ll[i] + 128 * (rowA[r] + colB[c]) -
           16384 * K;
  }
}

}  // namespace

int op_split16(const int16_t* src, uint64_t n, int8_t* hi, int8_t* lo, cudaStream_t s) {
  if (!n) return kOk;
  const uint64_t threads = (n + 7) / 8;
  k_split16<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(src, n, hi, lo);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

int op_igemm_combine(const int32_t* hh, const int32_t* hl, const int32_t* lh, const int32_t* ll,
                     const int64_t* rowA, const int64_t* colB, int64_t K, int64_t* C, int M,
                     int N, cudaStream_t s) {
  if (M <= 0 || N <= 0) return kOk;
  k_igemm_combine<<<grid_for((uint64_t)M * N, 256, 8), 256, 0, s>>>(hh, hl, lh, ll, rowA, colB,
                                                                     K, C, M, N);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

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
  // skinny products (few output tiles, long K): split K so the grid covers
  // about two waves of SMs, each slice a multiple of the 64-column K step
  int kslice = K;
  const int tiles = (int)(grid.x * grid.y);
  if (tiles < kSMs && K >= 2 * 256) {
    int splits = (2 * kSMs + tiles - 1) / tiles;
    const int max_splits = K / 256;
    if (splits > max_splits) splits = max_splits;
    kslice = (K + splits - 1) / splits;
    kslice = (kslice + kTK - 1) / kTK * kTK;
    grid.z = (K + kslice - 1) / kslice;
    ZKL_CUDA(cudaMemsetAsync(C, 0, (size_t)M * N * 8, s));
  }
  static bool attr = false;
  const size_t smem = 2 * kStage * sizeof(int16_t);
  if (!attr) {
    ZKL_CUDA(cudaFuncSetAttribute(k_igemm16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = true;
  }
  k_igemm16<<<grid, 256, smem, s>>>(A, B, C, M, K, N, kslice);
  ZKL_LAUNCH_CHECK();
  return kOk;
}

}  // namespace zkl
