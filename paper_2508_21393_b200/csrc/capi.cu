// extern "C" entry points (declared in include/zkl_b200.h): argument
// checking, canonical <-> Montgomery scalar conversion on the host, dispatch
// on the field id.
#include <vector>

#include "../../include/zkl_b200.h"
#include "ops.cuh"
#include "transcript.cuh"

using namespace zkl;

namespace zkl {
void prof_enable(bool on);
void prof_collect(int kind, double* ms, double* bytes, double* units, uint64_t* count);
}  // namespace zkl

namespace {

template <class F>
typename F::T scalar(const uint8_t* canon) {
  if (!canon) return F::zero();
  return load_canon<F>(canon);
}

template <class F>
Terms<F> make_terms(int degree, int nterms, const int32_t* nfactors, const int32_t* factors,
                    const uint8_t* coeffs, int k, int* err) {
  Terms<F> tm;
  *err = 0;
  tm.degree = degree;
  tm.nterms = nterms;
  for (int t = 0; t < kMaxTerms; t++) {
    tm.nf[t] = 0;
    tm.fi[t][0] = tm.fi[t][1] = tm.fi[t][2] = 0;
    tm.coef[t] = F::zero();
  }
  for (int t = 0; t < nterms; t++) {
    if (nfactors[t] < 0 || nfactors[t] > 3 || nfactors[t] > degree) *err = 1;
    tm.nf[t] = nfactors[t];
    for (int s = 0; s < nfactors[t] && s < 3; s++) {
      int f = factors[3 * t + s];
      if (f < 0 || f >= k) *err = 1;
      tm.fi[t][s] = f;
    }
    tm.coef[t] = load_canon<F>(coeffs + (size_t)t * F::kBytes);
  }
  return tm;
}

template <class F>
int sumcheck_round(void* const* tables, int k, uint64_t size, int fold, const uint8_t* r_prev,
                   int degree, int nterms, const int32_t* nfactors, const int32_t* factors,
                   const uint8_t* coeffs, const uint8_t* post_add, const uint8_t* post_mul,
                   uint8_t* evals_out, cudaStream_t s) {
  if (nterms < 0 || nterms > kMaxTerms) {
    set_error("sumcheck_round: %d terms (max %d)", nterms, kMaxTerms);
    return kErrArg;
  }
  int err;
  Terms<F> tm = make_terms<F>(degree, nterms, nfactors, factors, coeffs, k, &err);
  if (err) { set_error("sumcheck_round: bad term factors"); return kErrArg; }
  Post<F> post;
  post.add = scalar<F>(post_add);
  post.mul = post_mul ? scalar<F>(post_mul) : F::one();
  typename F::T r = fold ? scalar<F>(r_prev) : F::zero();
  return op_sumcheck_round<F>(tables, k, size, fold != 0, r, tm, post, evals_out, s);
}

template <class F>
int sumcheck_prove(void* const* tables, int k, int num_vars, int degree, int nterms,
                   const int32_t* nfactors, const int32_t* factors, const uint8_t* coeffs,
                   const uint8_t* post_add, const uint8_t* post_mul, uint8_t* state,
                   uint8_t* rounds_out, uint8_t* point_out, uint8_t* finals_out, cudaStream_t s) {
  if (nterms < 0 || nterms > kMaxTerms || num_vars < 0 || num_vars > 63) {
    set_error("sumcheck_prove: bad nterms/num_vars");
    return kErrArg;
  }
  int err;
  Terms<F> tm = make_terms<F>(degree, nterms, nfactors, factors, coeffs, k, &err);
  if (err) { set_error("sumcheck_prove: bad term factors"); return kErrArg; }
  std::vector<typename F::T> adds;
  if (post_add) {
    adds.resize(num_vars > 0 ? num_vars : 1);
    for (int j = 0; j < num_vars; j++) adds[j] = load_canon<F>(post_add + (size_t)j * F::kBytes);
  }
  typename F::T mul = post_mul ? scalar<F>(post_mul) : F::one();
  return op_sumcheck_prove<F>(tables, k, num_vars, tm, post_add ? adds.data() : nullptr, mul,
                              state, rounds_out, point_out, finals_out, s);
}

template <class F>
int sumcheck_prove_sharded(void* const* tables, int k, int num_vars, int degree, int nterms,
                           const int32_t* nfactors, const int32_t* factors, const uint8_t* coeffs,
                           const uint8_t* post_add, const uint8_t* post_mul, uint8_t* state,
                           uint8_t* rounds_out, uint8_t* point_out, uint8_t* finals_out,
                           cudaStream_t s) {
  if (nterms < 0 || nterms > kMaxTerms || num_vars < 0 || num_vars > 63 || k < 1 ||
      k > kMaxTables) {
    set_error("sumcheck_prove_sharded: bad nterms/num_vars/k");
    return kErrArg;
  }
  int err;
  Terms<F> tm = make_terms<F>(degree, nterms, nfactors, factors, coeffs, k, &err);
  if (err) { set_error("sumcheck_prove_sharded: bad term factors"); return kErrArg; }
  std::vector<typename F::T> adds;
  if (post_add) {
    adds.resize(num_vars > 0 ? num_vars : 1);
    for (int j = 0; j < num_vars; j++) adds[j] = load_canon<F>(post_add + (size_t)j * F::kBytes);
  }
  typename F::T mul = post_mul ? scalar<F>(post_mul) : F::one();
  return op_sumcheck_prove_sharded<F>(tables, k, num_vars, tm, post_add ? adds.data() : nullptr,
                                      mul, state, rounds_out, point_out, finals_out, s);
}

template <class F>
int transcript_challenge(uint8_t* state, const char* label, size_t llen, uint8_t* out) {
  HostTranscript tr;
  memcpy(tr.state, state, 64);
  uint8_t raw[64];
  tr.challenge_raw(label, llen, raw);
  reduce512<F>(raw, out);
  memcpy(state, tr.state, 64);
  return kOk;
}

template <class F>
int dot_impl(uint8_t* out, const void* a, const void* b, uint64_t n, cudaStream_t s) {
  void* ws;
  int rc = scratch_reserve(sizeof(typename F::T) * 2, &ws, s);
  if (rc) return rc;
  rc = op_dot<F>((typename F::T*)ws, a, b, n, s);
  if (rc) return rc;
  return op_read<F>(out, ws, 1, s);
}

}  // namespace

#define DISPATCH(field, EXPR_FR, EXPR_M61)                                      \
  do {                                                                          \
    if ((field) == ZKL_FIELD_BLS12_381_FR) { using F = Fr255; return EXPR_FR; }  \
    if ((field) == ZKL_FIELD_M61) { using F = M61; return EXPR_M61; }          \
    set_error("unknown field id %d", (int)(field));                             \
    return kErrArg;                                                             \
  } while (0)
#define D(field, EXPR) DISPATCH(field, EXPR, EXPR)

template <class F>
static int logup_tiled_impl(void* const* tables, int tile_log, int num_vars, int rounds,
                            const uint8_t* u_canon, const uint8_t* coeffs_canon, int flags,
                            uint8_t* state_inout, uint8_t* rounds_out, uint8_t* point_out,
                            void* stream) {
  using T = typename F::T;
  if (num_vars < 1 || num_vars > 63) {
    set_error("logup_tiled: bad num_vars");
    return kErrArg;
  }
  T c[5];
  for (int t = 0; t < 5; t++) c[t] = load_canon<F>(coeffs_canon + F::kBytes * t);
  std::vector<T> u(num_vars);
  for (int j = 0; j < num_vars; j++) u[j] = load_canon<F>(u_canon + (size_t)F::kBytes * j);
  return op_logup_tiled<F>(tables, tile_log, num_vars, rounds, u.data(), c, flags & 3,
                           state_inout, rounds_out, point_out, (cudaStream_t)stream);
}
extern "C" {

int zkl_abi_version(void) { return 3; }
uint64_t zkl_launch_count(void) { return g_launches; }
const char* zkl_last_error(void) { return get_error(); }
int zkl_elem_bytes(int field) {
  if (field == ZKL_FIELD_BLS12_381_FR) return 32;
  if (field == ZKL_FIELD_M61) return 8;
  return kErrArg;
}

int zkl_to_mont(int field, void* dst, const void* src, uint64_t n, void* stream) {
  D(field, op_to_mont<F>(dst, src, n, (cudaStream_t)stream));
}
int zkl_from_mont(int field, void* dst, const void* src, uint64_t n, void* stream) {
  D(field, op_from_mont<F>(dst, src, n, (cudaStream_t)stream));
}
int zkl_pair_combine(int field, void* dst, const void* x, int x_type, const void* y, int y_type,
                     uint64_t n, const uint8_t* alpha_canon, void* stream) {
  D(field, op_pair_combine<F>(dst, x, x_type, y, y_type, n, scalar<F>(alpha_canon),
                              (cudaStream_t)stream));
}
int zkl_lift(int field, int int_type, void* dst, const void* src, uint64_t n, void* stream) {
  D(field, op_lift<F>(dst, src, int_type, n, (cudaStream_t)stream));
}

static int eq_table_impl_fr(void* dst, const uint8_t* pt, int m, cudaStream_t s) {
  if (m < 0 || m > kMaxPoint) { set_error("eq_table: m=%d", m); return kErrArg; }
  Fr255::T p[kMaxPoint];
  for (int j = 0; j < m; j++) p[j] = load_canon<Fr255>(pt + 32 * j);
  return op_eq_table<Fr255>(dst, p, m, s);
}
static int eq_table_impl_m61(void* dst, const uint8_t* pt, int m, cudaStream_t s) {
  if (m < 0 || m > kMaxPoint) { set_error("eq_table: m=%d", m); return kErrArg; }
  M61::T p[kMaxPoint];
  for (int j = 0; j < m; j++) p[j] = load_canon<M61>(pt + 8 * j);
  return op_eq_table<M61>(dst, p, m, s);
}
int zkl_eq_table(int field, void* dst, const uint8_t* point_canon, int m, void* stream) {
  DISPATCH(field, eq_table_impl_fr(dst, point_canon, m, (cudaStream_t)stream),
           eq_table_impl_m61(dst, point_canon, m, (cudaStream_t)stream));
}

int zkl_fold(int field, void* dst, const void* src, uint64_t half, const uint8_t* r_canon,
             void* stream) {
  D(field, op_fold<F>(dst, src, half, scalar<F>(r_canon), (cudaStream_t)stream));
}
int zkl_axpy(int field, void* y, const void* a, const uint8_t* k_canon, const void* b, uint64_t n,
             void* stream) {
  D(field, op_axpy<F>(y, a, scalar<F>(k_canon), b, n, (cudaStream_t)stream));
}
int zkl_expand(int field, void* dst, uint64_t dst_n, const void* src, uint64_t src_n, int mode,
               const uint8_t* add_canon, const uint8_t* pad_canon, void* stream) {
  D(field, op_expand<F>(dst, dst_n, src, src_n, mode, scalar<F>(add_canon), scalar<F>(pad_canon),
                        (cudaStream_t)stream));
}
int zkl_lift_u32(int field, void* dst, const uint32_t* src, uint64_t n, void* stream) {
  D(field, op_lift_u32<F>(dst, src, n, (cudaStream_t)stream));
}
int zkl_read(int field, uint8_t* host_out, const void* src, uint64_t n, void* stream) {
  D(field, op_read<F>(host_out, src, n, (cudaStream_t)stream));
}

int zkl_dot(int field, uint8_t* out_host, const void* a, const void* b, uint64_t n, void* stream) {
  D(field, dot_impl<F>(out_host, a, b, n, (cudaStream_t)stream));
}

int zkl_sumcheck_round(int field, void* const* tables, int k, uint64_t size, int fold,
                       const uint8_t* r_prev_canon, int degree, int nterms,
                       const int32_t* nfactors, const int32_t* factors,
                       const uint8_t* coeffs_canon, const uint8_t* post_add_canon,
                       const uint8_t* post_mul_canon, uint8_t* evals_out_host, void* stream) {
  D(field, sumcheck_round<F>(tables, k, size, fold, r_prev_canon, degree, nterms, nfactors,
                             factors, coeffs_canon, post_add_canon, post_mul_canon,
                             evals_out_host, (cudaStream_t)stream));
}
int zkl_sumcheck_prove(int field, void* const* tables, int k, int num_vars, int degree,
                       int nterms, const int32_t* nfactors, const int32_t* factors,
                       const uint8_t* coeffs_canon, const uint8_t* post_add_canon,
                       const uint8_t* post_mul_canon, uint8_t* state_inout, uint8_t* rounds_out,
                       uint8_t* point_out, uint8_t* finals_out, void* stream) {
  D(field, sumcheck_prove<F>(tables, k, num_vars, degree, nterms, nfactors, factors,
                             coeffs_canon, post_add_canon, post_mul_canon, state_inout,
                             rounds_out, point_out, finals_out, (cudaStream_t)stream));
}
int zkl_sumcheck_prove_sharded(int field, void* const* tables, int k, int num_vars, int degree,
                               int nterms, const int32_t* nfactors, const int32_t* factors,
                               const uint8_t* coeffs_canon, const uint8_t* post_add_canon,
                               const uint8_t* post_mul_canon, uint8_t* state_inout,
                               uint8_t* rounds_out, uint8_t* point_out, uint8_t* finals_out,
                               void* stream) {
  D(field, sumcheck_prove_sharded<F>(tables, k, num_vars, degree, nterms, nfactors, factors,
                                     coeffs_canon, post_add_canon, post_mul_canon, state_inout,
                                     rounds_out, point_out, finals_out, (cudaStream_t)stream));
}
int zkl_igemm_i16(const int16_t* A, const int16_t* B, int64_t* C, int M, int K, int N,
                  void* stream) {
  return op_igemm16(A, B, C, M, K, N, (cudaStream_t)stream);
}
int zkl_split_i16(const int16_t* src, uint64_t n, int8_t* hi, int8_t* lo, void* stream) {
  return op_split16(src, n, hi, lo, (cudaStream_t)stream);
}
int zkl_igemm_combine(const int32_t* hh, const int32_t* hl, const int32_t* lh, const int32_t* ll,
                      const int64_t* rowA, const int64_t* colB, int64_t K, int64_t* C, int M,
                      int N, void* stream) {
  return op_igemm_combine(hh, hl, lh, ll, rowA, colB, K, C, M, N, (cudaStream_t)stream);
}
uint64_t zkl_commit_table_bytes(int group, int ngen) { return commit_table_bytes(group, ngen); }
int zkl_commit_tables(int group, const uint8_t* gens_canon, int ngen, void* tables, void* stream) {
  return op_commit_tables(group, gens_canon, ngen, tables, (cudaStream_t)stream);
}
int zkl_commit_rows(int group, const void* tables, int cols, const void* values,
                    const void* blinding, int blind_gen, int rows, uint8_t* rows_out,
                    void* stream) {
  return op_commit_rows(group, tables, cols, values, blinding, blind_gen, rows, rows_out,
                        (cudaStream_t)stream);
}
int zkl_shake256(const uint8_t* in, uint64_t len, uint8_t* out, uint64_t outlen) {
  shake256(in, (size_t)len, out, (size_t)outlen);
  return kOk;
}
int zkl_transcript_append(uint8_t* state_inout, const uint8_t* label, uint64_t label_len,
                          const uint8_t* data, uint64_t data_len) {
  HostTranscript tr;
  memcpy(tr.state, state_inout, 64);
  tr.append((const char*)label, (size_t)label_len, data, (size_t)data_len);
  memcpy(state_inout, tr.state, 64);
  return kOk;
}
int zkl_transcript_challenge(int field, uint8_t* state_inout, const uint8_t* label,
                             uint64_t label_len, uint8_t* out_canon) {
  D(field, transcript_challenge<F>(state_inout, (const char*)label, (size_t)label_len,
                                   out_canon));
}
int zkl_transcript_append_ints(uint8_t* state_inout, const uint8_t* label, uint64_t label_len,
                               const uint8_t* values, uint64_t count, uint64_t stride) {
  if (stride == 0 || stride > 64) {
    set_error("transcript_append_ints: bad stride %llu", (unsigned long long)stride);
    return kErrArg;
  }
  HostTranscript tr;
  memcpy(tr.state, state_inout, 64);
  for (uint64_t i = 0; i < count; i++) {
    const uint8_t* v = values + i * stride;
    size_t len = (size_t)stride;
    while (len > 1 && v[len - 1] == 0) len--;  // minimal little-endian, >= 1 byte
    tr.append((const char*)label, (size_t)label_len, v, len);
  }
  memcpy(state_inout, tr.state, 64);
  return kOk;
}
int zkl_transcript_challenge_vector(int field, uint8_t* state_inout, const uint8_t* label,
                                    uint64_t label_len, uint64_t count, uint8_t* out_canon) {
  // label bytes as given (any length, NULs included) + "/<i>"
  const size_t nb = field == ZKL_FIELD_M61 ? 8 : 32;
  std::vector<uint8_t> buf(label, label + label_len);
  for (uint64_t i = 0; i < count; i++) {
    char num[24];
    const int w = snprintf(num, sizeof(num), "/%llu", (unsigned long long)i);
    buf.resize(label_len);
    buf.insert(buf.end(), num, num + w);
    const int rc = zkl_transcript_challenge(field, state_inout, buf.data(), buf.size(),
                                            out_canon + i * nb);
    if (rc) return rc;
  }
  return kOk;
}
int zkl_sumcheck_finish(int field, void* const* tables, int k, const uint8_t* r_last_canon,
                        uint8_t* finals_out_host, void* stream) {
  D(field, op_sumcheck_finish<F>(tables, k, scalar<F>(r_last_canon), finals_out_host,
                                 (cudaStream_t)stream));
}
int zkl_batch_inverse(int field, void* dst, const void* src, uint64_t n, const uint8_t* add_canon,
                      int64_t* first_zero, void* stream) {
  D(field, op_batch_inverse<F>(dst, src, n, scalar<F>(add_canon), add_canon != nullptr,
                               first_zero, (cudaStream_t)stream));
}
int zkl_multiplicities(int field, const void* secret, uint64_t d, const void* table, uint64_t n,
                       uint32_t* counts, int64_t* first_miss, void* stream) {
  D(field, op_multiplicities<F>(secret, d, table, n, counts, first_miss, (cudaStream_t)stream));
}
int zkl_multiplicities_index(int field, const void* secret, uint64_t d, const void* table,
                             uint64_t n, uint32_t* counts, uint32_t* index_out,
                             int64_t* first_miss, void* stream) {
  D(field, op_multiplicities<F>(secret, d, table, n, counts, first_miss, (cudaStream_t)stream,
                                index_out));
}
int zkl_pair_multiplicities(int field, const void* x, int x_type, const void* y, int y_type,
                            uint64_t d, int64_t table_x0, const int32_t* table_y,
                            const void* secret, const void* table, uint64_t n, uint32_t* counts,
                            uint32_t* index_out, int64_t* first_miss, void* stream) {
  D(field, op_pair_multiplicities<F>(x, x_type, y, y_type, d, table_x0, table_y, secret, table, n,
                                     counts, index_out, first_miss, (cudaStream_t)stream));
}
int zkl_rescale_witness(const void* wide, int wide_type, uint64_t n, int64_t divisor,
                        int64_t lift, int64_t qmin, int64_t qmax, int16_t* q_out, int16_t* r_out,
                        int64_t* first_bad, uint64_t* n_bad, void* stream) {
  return op_rescale_witness(wide, wide_type, n, divisor, lift, qmin, qmax, q_out, r_out,
                            first_bad, n_bad, (cudaStream_t)stream);
}
int zkl_range_multiplicities(const void* x, int x_type, uint64_t d, int64_t table_x0,
                             uint64_t n, uint32_t* counts, uint32_t* index_out,
                             int64_t* first_miss, void* stream) {
  return op_range_multiplicities(x, x_type, d, table_x0, n, counts, index_out, first_miss,
                                 (cudaStream_t)stream);
}
int zkl_gather(int field, void* dst, const void* src, uint64_t src_n, const uint32_t* idx,
               uint64_t n, const uint8_t* add_canon, void* stream) {
  D(field, op_gather<F>(dst, src, src_n, idx, n, scalar<F>(add_canon), add_canon != nullptr,
                        (cudaStream_t)stream));
}
int zkl_matmul_prove(int field, int a_type, const void* A, int b_type, const void* B, int c_type,
                     const void* C, int d0, int d1, int d2, uint8_t* state_inout,
                     uint8_t* rounds_out, uint8_t* point_out, uint8_t* finals_out, void* stream) {
  D(field, op_matmul_prove<F>(a_type, A, b_type, B, c_type, C, d0, d1, d2, state_inout,
                              rounds_out, point_out, finals_out, (cudaStream_t)stream));
}
int zkl_matmul_prove_batch(int field, int nclaims, const int* types, const void* const* mats,
                           const int* dims, const uint8_t* pre, const uint64_t* pre_off,
                           uint8_t* state_inout, uint8_t* rounds_out, uint8_t* point_out,
                           uint8_t* finals_out, void* stream) {
  D(field, op_matmul_prove_batch<F>(nclaims, types, mats, dims, pre, pre_off, state_inout,
                                    rounds_out, point_out, finals_out, (cudaStream_t)stream));
}
int zkl_logup_tiled_rounds(int field, void* const* tables, int tile_log, int num_vars, int rounds,
                           const uint8_t* u_canon, const uint8_t* coeffs_canon, int flags,
                           uint8_t* state_inout, uint8_t* rounds_out, uint8_t* point_out,
                           void* stream) {
  D(field, logup_tiled_impl<F>(tables, tile_log, num_vars, rounds, u_canon, coeffs_canon, flags,
                               state_inout, rounds_out, point_out, stream));
}
int zkl_prof_enable(int on) {
  zkl::prof_enable(on != 0);
  return kOk;
}
int zkl_prof_collect(int kind, double* ms, double* bytes, double* units, uint64_t* count) {
  if (kind < 0 || kind >= kProfKinds) {
    set_error("prof_collect: bad kind %d", kind);
    return kErrArg;
  }
  zkl::prof_collect(kind, ms, bytes, units, count);
  return kOk;
}
int zkl_matvec(int field, int mtype, const void* M, uint64_t rows, uint64_t cols, int transpose,
               const void* x, void* y, void* stream) {
  D(field, op_matvec<F>(mtype, M, rows, cols, transpose, x, y, (cudaStream_t)stream));
}

}  // extern "C"
