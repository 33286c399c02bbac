// Integer-matrix x field-vector products for the factored zkMat prover.
//
// Reference context: the zkMat claim of gadgets.py:210-251 is proven without
// materialising its 2^(d0+d1+d2) replicated tables; instead every MLE partial
// evaluation it needs is a matrix-vector product against an eq-vector:
//   B E_v, C E_v, A (B E_v)   (row products,  y = M x)
//   E_rho_u^T A, E_rho_u^T C, E_rho_w^T B   (column products, y = M^T x)
// (derivation: DESIGN.md "Factored zkMat").
//
// Fr255 with integer matrices (int16 / int32 / int64): multiply-accumulate
// into a wide (320/384-bit) integer accumulator with one 16-IMAD row of
// mad.lo/hi.cc per 32-bit matrix word and no modular reduction in the inner
// loop.  Signed entries use offset binary: sum (s + o) x - o * sum x, so the
// inner loop is unsigned; the wide sum is reduced mod p once per output.
// Other combinations (M61, field-valued matrices) multiply-add in the field.
#include "ops.cuh"

namespace zkl {

// ---------------------------------------------------------------------------
// wide accumulator (Fr255)
template <int W>
struct Wide {
  uint32_t w[W];
};

// a[0..9] += u * x  (10-limb accumulator)
ZKL_D void mac10(Wide<10>& a, uint32_t u, const fr_t& x) {
  asm("mad.lo.cc.u32  %0, %10, %18, %0;\n\t"
      "madc.lo.cc.u32 %1, %11, %18, %1;\n\t"
      "madc.lo.cc.u32 %2, %12, %18, %2;\n\t"
      "madc.lo.cc.u32 %3, %13, %18, %3;\n\t"
      "madc.lo.cc.u32 %4, %14, %18, %4;\n\t"
      "madc.lo.cc.u32 %5, %15, %18, %5;\n\t"
      "madc.lo.cc.u32 %6, %16, %18, %6;\n\t"
      "madc.lo.cc.u32 %7, %17, %18, %7;\n\t"
      "addc.cc.u32    %8, %8, 0;\n\t"
      "addc.u32       %9, %9, 0;\n\t"
      "mad.hi.cc.u32  %1, %10, %18, %1;\n\t"
      "madc.hi.cc.u32 %2, %11, %18, %2;\n\t"
      "madc.hi.cc.u32 %3, %12, %18, %3;\n\t"
      "madc.hi.cc.u32 %4, %13, %18, %4;\n\t"
      "madc.hi.cc.u32 %5, %14, %18, %5;\n\t"
      "madc.hi.cc.u32 %6, %15, %18, %6;\n\t"
      "madc.hi.cc.u32 %7, %16, %18, %7;\n\t"
      "madc.hi.cc.u32 %8, %17, %18, %8;\n\t"
      "addc.u32       %9, %9, 0;\n\t"
      : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]), "+r"(a.w[5]),
        "+r"(a.w[6]), "+r"(a.w[7]), "+r"(a.w[8]), "+r"(a.w[9])
      : "r"(x.v[0]), "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]),
        "r"(x.v[6]), "r"(x.v[7]), "r"(u));
}

// a[off..off+9] += u * x for a 12-limb accumulator, off in {0, 1}
template <int OFF>
ZKL_D void mac12(Wide<12>& a, uint32_t u, const fr_t& x) {
  uint32_t* w = a.w + OFF;
  if (OFF == 0) {
    asm("mad.lo.cc.u32  %0, %12, %20, %0;\n\t"
        "madc.lo.cc.u32 %1, %13, %20, %1;\n\t"
        "madc.lo.cc.u32 %2, %14, %20, %2;\n\t"
        "madc.lo.cc.u32 %3, %15, %20, %3;\n\t"
        "madc.lo.cc.u32 %4, %16, %20, %4;\n\t"
        "madc.lo.cc.u32 %5, %17, %20, %5;\n\t"
        "madc.lo.cc.u32 %6, %18, %20, %6;\n\t"
        "madc.lo.cc.u32 %7, %19, %20, %7;\n\t"
        "addc.cc.u32    %8, %8, 0;\n\t"
        "addc.cc.u32    %9, %9, 0;\n\t"
        "addc.cc.u32    %10, %10, 0;\n\t"
        "addc.u32       %11, %11, 0;\n\t"
        "mad.hi.cc.u32  %1, %12, %20, %1;\n\t"
        "madc.hi.cc.u32 %2, %13, %20, %2;\n\t"
        "madc.hi.cc.u32 %3, %14, %20, %3;\n\t"
        "madc.hi.cc.u32 %4, %15, %20, %4;\n\t"
        "madc.hi.cc.u32 %5, %16, %20, %5;\n\t"
        "madc.hi.cc.u32 %6, %17, %20, %6;\n\t"
        "madc.hi.cc.u32 %7, %18, %20, %7;\n\t"
        "madc.hi.cc.u32 %8, %19, %20, %8;\n\t"
        "addc.cc.u32    %9, %9, 0;\n\t"
        "addc.cc.u32    %10, %10, 0;\n\t"
        "addc.u32       %11, %11, 0;\n\t"
        : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]),
          "+r"(w[7]), "+r"(w[8]), "+r"(w[9]), "+r"(w[10]), "+r"(w[11])
        : "r"(x.v[0]), "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]),
          "r"(x.v[6]), "r"(x.v[7]), "r"(u));
  } else {
    asm("mad.lo.cc.u32  %0, %11, %19, %0;\n\t"
        "madc.lo.cc.u32 %1, %12, %19, %1;\n\t"
        "madc.lo.cc.u32 %2, %13, %19, %2;\n\t"
        "madc.lo.cc.u32 %3, %14, %19, %3;\n\t"
        "madc.lo.cc.u32 %4, %15, %19, %4;\n\t"
        "madc.lo.cc.u32 %5, %16, %19, %5;\n\t"
        "madc.lo.cc.u32 %6, %17, %19, %6;\n\t"
        "madc.lo.cc.u32 %7, %18, %19, %7;\n\t"
        "addc.cc.u32    %8, %8, 0;\n\t"
        "addc.cc.u32    %9, %9, 0;\n\t"
        "addc.u32       %10, %10, 0;\n\t"
        "mad.hi.cc.u32  %1, %11, %19, %1;\n\t"
        "madc.hi.cc.u32 %2, %12, %19, %2;\n\t"
        "madc.hi.cc.u32 %3, %13, %19, %3;\n\t"
        "madc.hi.cc.u32 %4, %14, %19, %4;\n\t"
        "madc.hi.cc.u32 %5, %15, %19, %5;\n\t"
        "madc.hi.cc.u32 %6, %16, %19, %6;\n\t"
        "madc.hi.cc.u32 %7, %17, %19, %7;\n\t"
        "madc.hi.cc.u32 %8, %18, %19, %8;\n\t"
        "addc.cc.u32    %9, %9, 0;\n\t"
        "addc.u32       %10, %10, 0;\n\t"
        : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]),
          "+r"(w[7]), "+r"(w[8]), "+r"(w[9]), "+r"(w[10])
        : "r"(x.v[0]), "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]),
          "r"(x.v[6]), "r"(x.v[7]), "r"(u));
  }
}

// X = lo + hi 2^256 (hi < 2^128) -> X mod p in Montgomery form (X already
// carries the factor R through x, so plain reduction mod p is what we want).
template <int W>
ZKL_D fr_t reduce_wide(const Wide<W>& a) {
  fr_t lo, hi = Fr255::zero();
#pragma unroll
  for (int i = 0; i < 8; i++) lo.v[i] = a.w[i];
#pragma unroll
  for (int i = 8; i < W; i++) hi.v[i - 8] = a.w[i];
  lo = Fr255::reduce_once(Fr255::reduce_once(lo));  // lo < 2^256 < 3p
  hi = Fr255::mul(hi, Fr255::r2());                 // hi * 2^256 mod p
  return Fr255::add(lo, hi);
}

// ---------------------------------------------------------------------------
// accumulation policies
struct AccI16 {  // Fr255, int16 entries, offset 2^15
  using M = int16_t;
  Wide<10> a;
  ZKL_D void init() {
#pragma unroll
    for (int i = 0; i < 10; i++) a.w[i] = 0;
  }
  ZKL_D void mac(int16_t s, const fr_t& x) { mac10(a, (uint32_t)((int32_t)s + 32768), x); }
  ZKL_D fr_t done() const { return reduce_wide<10>(a); }
  ZKL_D static fr_t offset() { return Fr255::from_u32(1u << 15); }
};
struct AccI32 {  // Fr255, int32 entries, offset 2^31
  using M = int32_t;
  Wide<10> a;
  ZKL_D void init() {
#pragma unroll
    for (int i = 0; i < 10; i++) a.w[i] = 0;
  }
  ZKL_D void mac(int32_t s, const fr_t& x) { mac10(a, (uint32_t)s ^ 0x80000000u, x); }
  ZKL_D fr_t done() const { return reduce_wide<10>(a); }
  ZKL_D static fr_t offset() { return Fr255::from_u32(1u << 31); }
};
struct AccI64 {  // Fr255, int64 entries, offset 2^63
  using M = int64_t;
  Wide<12> a;
  ZKL_D void init() {
#pragma unroll
    for (int i = 0; i < 12; i++) a.w[i] = 0;
  }
  ZKL_D void mac(int64_t s, const fr_t& x) {
    uint64_t u = (uint64_t)s ^ 0x8000000000000000ull;
    mac12<0>(a, (uint32_t)u, x);
    mac12<1>(a, (uint32_t)(u >> 32), x);
  }
  ZKL_D fr_t done() const { return reduce_wide<12>(a); }
  ZKL_D static fr_t offset() {
    return Fr255::mul(Fr255::from_u32(1u << 31), Fr255::from_i64(1ll << 32));
  }
};
template <class F, class I>
struct AccField {  // generic: acc += lift(s) * x in the field
  using M = I;
  typename F::T a;
  ZKL_D void init() { a = F::zero(); }
  ZKL_D void mac(I s, const typename F::T& x) { a = F::add(a, F::mul(F::from_i64((int64_t)s), x)); }
  ZKL_D typename F::T done() const { return a; }
  ZKL_D static typename F::T offset() { return F::zero(); }
};
template <class F>
struct AccElem {  // field-valued matrix
  using M = typename F::T;
  typename F::T a;
  ZKL_D void init() { a = F::zero(); }
  ZKL_D void mac(const typename F::T& s, const typename F::T& x) { a = F::add(a, F::mul(s, x)); }
  ZKL_D typename F::T done() const { return a; }
  ZKL_D static typename F::T offset() { return F::zero(); }
};

// ---------------------------------------------------------------------------
// y[r] = sum_c M[r, c] x[c] - off * S,  S = sum_c x[c];  one warp per row
template <class F, class ACC>
__global__ void __launch_bounds__(256)
    k_rowmv(const typename ACC::M* M, uint64_t rows, uint64_t cols, const typename F::T* x,
            const typename F::T* S, typename F::T* y) {
  using T = typename F::T;
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const T corr = F::mul(*S, ACC::offset());
  for (uint64_t r = warp; r < rows; r += nwarps) {
    ACC acc;
    acc.init();
    const typename ACC::M* row = M + r * cols;
    for (uint64_t c = lane; c < cols; c += 32) acc.mac(row[c], x[c]);
    T f = warp_sum<F>(acc.done());
    if (lane == 0) y[r] = F::sub(f, corr);
  }
}

// column products: partial[by][c] = sum_{r in chunk by} x[r] M[r, c]
template <class F, class ACC>
__global__ void __launch_bounds__(256)
    k_colmv_part(const typename ACC::M* M, uint64_t rows, uint64_t cols, const typename F::T* x,
                 int cw, uint64_t rch, typename F::T* part) {
  using T = typename F::T;
  __shared__ T sm[256];
  const int tc = threadIdx.x % cw, rg = threadIdx.x / cw, ngrp = blockDim.x / cw;
  const uint64_t c = blockIdx.x * (uint64_t)cw + tc;
  const uint64_t r0 = blockIdx.y * rch;
  uint64_t r1 = r0 + rch;
  if (r1 > rows) r1 = rows;
  ACC acc;
  acc.init();
  if (c < cols)
    for (uint64_t r = r0 + rg; r < r1; r += ngrp) acc.mac(M[r * cols + c], x[r]);
  sm[threadIdx.x] = acc.done();
  __syncthreads();
  if (rg == 0 && c < cols) {
    T v = sm[tc];
    for (int g = 1; g < ngrp; g++) v = F::add(v, sm[g * cw + tc]);
    part[blockIdx.y * cols + c] = v;
  }
}

template <class F, class ACC>
__global__ void k_colmv_sum(const typename F::T* part, uint64_t nchunks, uint64_t cols,
                            const typename F::T* S, typename F::T* y) {
  using T = typename F::T;
  const T corr = F::mul(*S, ACC::offset());
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < cols;
       c += (uint64_t)gridDim.x * blockDim.x) {
    T v = F::zero();
    for (uint64_t b = 0; b < nchunks; b++) v = F::add(v, part[b * cols + c]);
    y[c] = F::sub(v, corr);
  }
}

template <class F, class ACC>
static int matvec_impl(const void* Mv, uint64_t rows, uint64_t cols, int transpose,
                       const void* xv, void* yv, cudaStream_t s) {
  using T = typename F::T;
  const auto* M = (const typename ACC::M*)Mv;
  const T* x = (const T*)xv;
  T* y = (T*)yv;
  uint64_t xlen = transpose ? rows : cols;
  // scratch: S (1) + partials
  int cw = 1;
  while (cw < 256 && (uint64_t)cw < cols) cw <<= 1;
  uint64_t col_blocks = (cols + cw - 1) / cw;
  uint64_t ngrp = 256 / cw;
  uint64_t want_rb = (4ull * kSMs + col_blocks - 1) / col_blocks;
  uint64_t max_rb = (rows + ngrp - 1) / ngrp;
  uint64_t rb = want_rb < max_rb ? want_rb : max_rb;
  if (rb < 1) rb = 1;
  if (rb > 65535) rb = 65535;
  uint64_t rch = (rows + rb - 1) / rb;
  rb = (rows + rch - 1) / rch;
  size_t need = sizeof(T) * (1 + (transpose ? rb * cols : 0)) + 64;
  void* ws;
  int rc = scratch_reserve(need, &ws, s);
  if (rc) return rc;
  T* S = (T*)ws;
  T* part = S + 1;
  rc = op_dot<F>(S, x, nullptr, xlen, s);
  if (rc) return rc;
  if (!transpose) {
    unsigned grid = grid_for(rows * 32, 256, 8);
    k_rowmv<F, ACC><<<grid, 256, 0, s>>>(M, rows, cols, x, S, y);
  } else {
    dim3 g((unsigned)col_blocks, (unsigned)rb);
    k_colmv_part<F, ACC><<<g, 256, 0, s>>>(M, rows, cols, x, cw, rch, part);
    ZKL_LAUNCH_CHECK();
    k_colmv_sum<F, ACC><<<grid_for(cols, 256), 256, 0, s>>>(part, rb, cols, S, y);
  }
  ZKL_LAUNCH_CHECK();
  return kOk;
}

template <class F>
int op_matvec(int mtype, const void* M, uint64_t rows, uint64_t cols, int transpose,
              const void* x, void* y, cudaStream_t s) {
  if (!rows || !cols) { set_error("matvec: empty matrix"); return kErrArg; }
  if constexpr (F::kId == Fr255::kId) {
    switch (mtype) {
      case 0: return matvec_impl<F, AccElem<F>>(M, rows, cols, transpose, x, y, s);
      case 1: return matvec_impl<F, AccI16>(M, rows, cols, transpose, x, y, s);
      case 2: return matvec_impl<F, AccI32>(M, rows, cols, transpose, x, y, s);
      case 3: return matvec_impl<F, AccI64>(M, rows, cols, transpose, x, y, s);
    }
  } else {
    switch (mtype) {
      case 0: return matvec_impl<F, AccElem<F>>(M, rows, cols, transpose, x, y, s);
      case 1: return matvec_impl<F, AccField<F, int16_t>>(M, rows, cols, transpose, x, y, s);
      case 2: return matvec_impl<F, AccField<F, int32_t>>(M, rows, cols, transpose, x, y, s);
      case 3: return matvec_impl<F, AccField<F, int64_t>>(M, rows, cols, transpose, x, y, s);
    }
  }
  set_error("matvec: bad matrix type %d", mtype);
  return kErrArg;
}

template int op_matvec<Fr255>(int, const void*, uint64_t, uint64_t, int, const void*, void*,
                              cudaStream_t);
template int op_matvec<M61>(int, const void*, uint64_t, uint64_t, int, const void*, void*,
                            cudaStream_t);

}  // namespace zkl
