// Host-side launchers (templated on the field), dispatched by capi.cu.
#pragma once
#include "common.cuh"

namespace zkl {

constexpr int kMaxTables = 8;
constexpr int kMaxTerms = 8;
constexpr int kMaxPoint = 64;

// element-wise ---------------------------------------------------------------
template <class F> int op_to_mont(void* dst, const void* src, uint64_t n, cudaStream_t s);
template <class F> int op_from_mont(void* dst, const void* src, uint64_t n, cudaStream_t s);
// mtype: 1 = int16, 2 = int32, 3 = int64 (signed; negatives -> p - |x|)
template <class F> int op_lift(void* dst, const void* src, int mtype, uint64_t n, cudaStream_t s);
// dst[i] = x[i] + alpha * y[i], signed integer columns (types 1..3 = int16/32/64)
template <class F>
int op_pair_combine(void* dst, const void* x, int tx, const void* y, int ty, uint64_t n,
                    typename F::T alpha, cudaStream_t s);
template <class F>
int op_eq_table(void* dst, const typename F::T* point, int m, cudaStream_t s);
// an eq point as kernels take it: r and 1 - r in storage form
template <class F>
struct PointArg {
  typename F::T r[kMaxPoint];
  typename F::T omr[kMaxPoint];
};
// eq table from a point in mapped host memory (m <= 16), staged through
// device slot slot_id (0..7; concurrent tables take different slots)
template <class F>
int op_eq_table_dev(void* dst, const PointArg<F>* pt_dev, int m, int slot_id, cudaStream_t s);
template <class F>
int op_fold(void* dst, const void* src, uint64_t half, typename F::T r, cudaStream_t s);
// y = a + k * b
template <class F>
int op_axpy(void* y, const void* a, typename F::T k, const void* b, uint64_t n, cudaStream_t s);
template <class F>
int op_mul(void* dst, const void* a, const void* b, uint64_t n, cudaStream_t s);
// canonical host copy of n device elements (synchronises)
template <class F> int op_read(uint8_t* host, const void* src, uint64_t n, cudaStream_t s);
// out = sum_i a[i]*b[i] (b == nullptr: sum_i a[i]); device scalar (Montgomery)
template <class F>
int op_dot(typename F::T* out_dev, const void* a, const void* b, uint64_t n, cudaStream_t s);

template <class F>
int op_expand(void* dst, uint64_t dst_n, const void* src, uint64_t src_n, int mode,
              typename F::T add, typename F::T pad, cudaStream_t s);
template <class F> int op_lift_u32(void* dst, const uint32_t* src, uint64_t n, cudaStream_t s);

// sumcheck -----------------------------------------------------------------------
template <class F>
struct Terms {
  int nterms;
  int degree;
  int nf[kMaxTerms];
  int fi[kMaxTerms][3];
  typename F::T coef[kMaxTerms];
  int tile_log;  // LOGUP_TILED: log2 of the table side's size (the low index bits)
  int inv_pair;  // LOGUP_TILED: A = 1/S entrywise before the first fold
  // LOGUP_TILED, indexed: the secret-side columns are never gathered.  Entry i
  // of A / S+beta is side_a / side_s[sidx[i]] (the table side, indexed by the
  // multiplicity histogram's query -> table index) until the first fold has
  // written them; rounds 0 and 1 (half == sidx_d / 4) read through sidx.
  const uint32_t* sidx;
  const typename F::T* side_a;
  const typename F::T* side_s;
  uint64_t sidx_d;
  uint64_t tiled_d;  // LOGUP_TILED: 2^num_vars (round 1 = the first fold: half * 4 == tiled_d)
};
template <class F>
struct Post {
  typename F::T add;  // evals[x] = mul * (sum_x + add)
  typename F::T mul;
};
template <class F>
int op_sumcheck_round(void* const* tables, int k, uint64_t size, bool fold,
                      typename F::T r_prev, const Terms<F>& terms, const Post<F>& post,
                      uint8_t* evals_host, cudaStream_t s);
template <class F>
int op_sumcheck_prove(void* const* tables, int k, int num_vars, const Terms<F>& tm,
                      const typename F::T* post_add, const typename F::T& post_mul,
                      uint8_t* state, uint8_t* rounds_out, uint8_t* point_out,
                      uint8_t* finals_out, cudaStream_t s);
template <class F>
int op_sumcheck_prove_sharded(void* const* tables, int k, int num_vars, const Terms<F>& tm,
                      const typename F::T* post_add, const typename F::T& post_mul,
                      uint8_t* state, uint8_t* rounds_out, uint8_t* point_out,
                      uint8_t* finals_out, cudaStream_t s);
int op_igemm16(const int16_t* A, const int16_t* B, int64_t* C, int M, int K, int N,
               cudaStream_t s);
int op_split16(const int16_t* src, uint64_t n, int8_t* hi, int8_t* lo, cudaStream_t s);
// Hyrax row commitments (commit.cu): group 0 = q 96 p + 1, 1 = q 52 (2^61-1) + 1
size_t commit_table_bytes(int group, int ngen);
int op_commit_tables(int group, const uint8_t* gens_canon, int ngen, void* tables,
                     cudaStream_t s);
int op_commit_rows(int group, const void* tables, int cols, const void* vals, const void* blind,
                   int blind_gen, int rows, uint8_t* out_canon, cudaStream_t s);
int op_igemm_combine(const int32_t* hh, const int32_t* hl, const int32_t* lh, const int32_t* ll,
                     const int64_t* rowA, const int64_t* colB, int64_t K, int64_t* C, int M,
                     int N, cudaStream_t s);
int shard_world();
int shard_rank();
int shard_exchange(const void* mine, size_t nbytes, uint8_t* out);
template <class F>
int op_sumcheck_finish(void* const* tables, int k, typename F::T r, uint8_t* finals_host,
                       cudaStream_t s);

// batch inversion: dst[i] = 1 / (src[i] + add); returns kErrZero and sets
// *first_zero to the first zero index when some src[i] + add == 0.
template <class F>
int op_batch_inverse(void* dst, const void* src, uint64_t n, typename F::T add, bool has_add,
                     int64_t* first_zero, cudaStream_t s);

// multiplicities ---------------------------------------------------------------
template <class F>
int op_multiplicities(const void* secret, uint64_t d, const void* table, uint64_t n,
                      uint32_t* counts, int64_t* first_miss, cudaStream_t s,
                      uint32_t* index_out = nullptr);
int op_rescale_witness(const void* wide, int wide_type, uint64_t n, int64_t divisor, int64_t lift,
                       int64_t qmin, int64_t qmax, int16_t* q_out, int16_t* r_out, int64_t* first_bad, uint64_t* n_bad, cudaStream_t s);
int op_range_multiplicities(const void* x, int xt, uint64_t d, int64_t x0, uint64_t n,
                            uint32_t* counts, uint32_t* index_out, int64_t* first_miss,
                            cudaStream_t s);
template <class F>
int op_pair_multiplicities(const void* x, int xt, const void* y, int yt, uint64_t d, int64_t x0,
                           const int32_t* ty, const void* secret, const void* table, uint64_t n,
                           uint32_t* counts, uint32_t* index_out, int64_t* first_miss,
                           cudaStream_t s);
template <class F>
int op_gather(void* dst, const void* src, uint64_t src_n, const uint32_t* idx, uint64_t n,
              typename F::T add, bool has_add, cudaStream_t s);

// matrix x field-vector ------------------------------------------------------------
// mtype: 0 = field (Montgomery), 1 = int16, 2 = int32, 3 = int64
template <class F>
int op_matvec(int mtype, const void* M, uint64_t rows, uint64_t cols, int transpose,
              const void* x, void* y, cudaStream_t s);

// replicated logUp claim, first rounds with the tiled evaluator (persistent.cu)
template <class F>
int op_logup_tiled(void* const* tables, int tile_log, int num_vars, int rounds,
                   const typename F::T* u, const typename F::T* coefs, int inv_pair,
                   uint8_t* state, uint8_t* rounds_out, uint8_t* point_out, cudaStream_t s);

// native zkMat driver (zkmat.cu): gadgets.py:241-251, factored
template <class F>
int op_matmul_prove(int ta, const void* A, int tb, const void* B, int tc, const void* C, int d0,
                    int d1, int d2, uint8_t* state, uint8_t* rounds_out, uint8_t* point_out,
                    uint8_t* finals_out, cudaStream_t s);
template <class F>
int op_matmul_prove_batch(int nclaims, const int* types, const void* const* mats, const int* dims,
                          const uint8_t* pre, const uint64_t* pre_off, uint8_t* state,
                          uint8_t* rounds_out, uint8_t* point_out, uint8_t* finals_out,
                          cudaStream_t s);

}  // namespace zkl
