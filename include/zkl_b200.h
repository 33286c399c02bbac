/*
 * zkl_b200 — C ABI of the B200-native zkLoRA sumcheck / logUp prover backend.
 *
 * Plain pointers and sizes only.  Device buffers are caller-owned (the Python
 * host allocates them with torch); `stream` is a cudaStream_t (NULL = legacy
 * default stream).  Field elements live on the device in the backend's
 * storage form: 32-byte Montgomery (field 0, BLS12-381 Fr) or 8-byte
 * canonical (field 1, 2^61-1), little-endian.  Every field SCALAR crossing
 * the ABI on the host side is canonical little-endian (32 or 8 bytes), like
 * the reference's field.to_bytes (pkg/src/zklora/field.py:58-60).
 *
 * Status: 0 ok; <0 error (zkl_last_error() describes it).  Error codes that
 * map to reference exceptions:
 *   ZKL_ERR_ZERO    -> zklora.field.InversionOfZero   (field.py:27-28, 38-39)
 *   ZKL_ERR_MISSING -> zklora.lookup.ElementNotInTable (lookup.py:94-98)
 * with the FIRST offending index written to the int64 out-parameter.
 *
 * Threading: the transcript is single-owner.  One host thread
 * proves on a device at a time: the per-device scratch arenas, mailbox and
 * the zkMat side stream are shared by the calls on that device.
 *
 * Each entry point names the reference interface it replaces.
 */
#ifndef ZKL_B200_H
#define ZKL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZKL_FIELD_BLS12_381_FR 0 /* field.py:9  MODULUS      */
#define ZKL_FIELD_M61 1          /* field.py:12 TEST_MODULUS */

#define ZKL_OK 0
#define ZKL_ERR_CUDA -1
#define ZKL_ERR_ARG -2
#define ZKL_ERR_ZERO -3
#define ZKL_ERR_MISSING -4
#define ZKL_ERR_UNSUPPORTED -5

/* matrix / integer element types */
#define ZKL_MT_FIELD 0
#define ZKL_MT_I16 1
#define ZKL_MT_I32 2
#define ZKL_MT_I64 3

int zkl_abi_version(void);
const char* zkl_last_error(void);
/* number of CUDA kernels this library has launched in this process */
uint64_t zkl_launch_count(void);
/* bytes per stored element (32 or 8); <0 for an unknown field */
int zkl_elem_bytes(int field);

/* canonical residues -> storage form and back (in place allowed).
 * Replaces the implicit int residues of field.py / quantize.py:176-183. */
int zkl_to_mont(int field, void* dst, const void* src, uint64_t n, void* stream);
int zkl_from_mont(int field, void* dst, const void* src, uint64_t n, void* stream);

/* signed int16/32/64 -> field (negatives as p-|x|): field.py:54-55
 * (from_signed) as used by QuantizedTensor.from_field, quantize.py:176-183. */
int zkl_lift(int field, int int_type, void* dst, const void* src, uint64_t n, void* stream);

/* Pair-table compression of a two-column lookup (gadgets.py:659-666 for the
 * secret, tables.py:131-140 for the table): dst[i] = x[i] + alpha * y[i]
 * mod p for signed integer columns x, y (ZKL_MT_I16 / I32 / I64). */
int zkl_pair_combine(int field, void* dst, const void* x, int x_type, const void* y, int y_type,
                     uint64_t n, const uint8_t* alpha_canon, void* stream);

/* eq(point, .) over {0,1}^m, point[0] = MSB: mle.py:67-82 (eq_table).
 * point_canon: m canonical scalars (host). */
int zkl_eq_table(int field, void* dst, const uint8_t* point_canon, int m, void* stream);

/* fold_table: dst[i] = (1-r) src[i] + r src[i+half], mle.py:50-56. */
int zkl_fold(int field, void* dst, const void* src, uint64_t half, const uint8_t* r_canon,
             void* stream);

/* y = a + k*b (device vectors, k host canonical). */
int zkl_axpy(int field, void* y, const void* a, const uint8_t* k_canon, const void* b, uint64_t n,
             void* stream);

/* Lifted logUp columns (lookup.py:188-202):
 *   mode 0 (pad):  dst[i] = i < src_n ? (src ? src[i] : 0) + add : pad
 *   mode 1 (tile): dst[i] = (src ? src[i % src_n] : 0) + add
 * add/pad canonical host scalars (NULL = 0). */
int zkl_expand(int field, void* dst, uint64_t dst_n, const void* src, uint64_t src_n, int mode,
               const uint8_t* add_canon, const uint8_t* pad_canon, void* stream);

/* uint32 counts (zkl_multiplicities output) -> field vector. */
int zkl_lift_u32(int field, void* dst, const uint32_t* src, uint64_t n, void* stream);

/* canonical host copy of n device elements (synchronises). */
int zkl_read(int field, uint8_t* host_out, const void* src, uint64_t n, void* stream);

/* out_host = sum_i a[i]*b[i] (b NULL: sum_i a[i]) as a canonical scalar. */
int zkl_dot(int field, uint8_t* out_host, const void* a, const void* b, uint64_t n, void* stream);

/* One round of prove_sumcheck (sumcheck.py:110-129):
 *   tables: k device pointers (host array), each holding `size` elements.
 *   fold != 0: first fold every table in place by r_prev (the previous
 *   round's challenge, sumcheck.py:129), then evaluate over the folded
 *   tables (size/2 entries); fold == 0: evaluate over `size` entries.
 *   evals_out_host[x] = post_mul * (post_add + sum_i combine(terms, t_x(i)))
 *   for x = 0..degree (combine: sumcheck.py:70-78; the claim's own rounds use
 *   post_add = 0, post_mul = 1).  Terms: nterms <= 8, nfactors[t] <= 3,
 *   factors[3*t + s] table indices, coeffs canonical (nterms scalars).
 *   Synchronises the stream (the transcript needs the evaluations). */
int zkl_sumcheck_round(int field, void* const* tables, int k, uint64_t size, int fold,
                       const uint8_t* r_prev_canon, int degree, int nterms,
                       const int32_t* nfactors, const int32_t* factors,
                       const uint8_t* coeffs_canon, const uint8_t* post_add_canon,
                       const uint8_t* post_mul_canon, uint8_t* evals_out_host, void* stream);

/* The whole of prove_sumcheck after _absorb_claim (sumcheck.py:108-130) with
 * the native transcript: state_inout is the 64-byte transcript state
 * (transcript.py:24-42), updated in place.  Per round: fused fold+eval, the
 * (degree+1) evaluations appended under b"sumcheck/eval" (minimal LE ints),
 * challenge b"sumcheck/round".  post_add_canon: num_vars scalars (one per
 * round) or NULL; post_mul_canon: NULL = 1.  Outputs (canonical LE):
 * rounds_out num_vars*(degree+1) scalars, point_out num_vars, finals_out k.
 * The tables are consumed: the last rounds of a claim may run on the host
 * (ZKL_HOST_TAIL), so their device contents afterwards are unspecified. */
int zkl_sumcheck_prove(int field, void* const* tables, int k, int num_vars, int degree,
                       int nterms, const int32_t* nfactors, const int32_t* factors,
                       const uint8_t* coeffs_canon, const uint8_t* post_add_canon,
                       const uint8_t* post_mul_canon, uint8_t* state_inout, uint8_t* rounds_out,
                       uint8_t* point_out, uint8_t* finals_out, void* stream);

/* Multi-GPU (ranks = processes of one node, one GPU each).
 * zkl_shard_open joins the rank set `name` (POSIX shared memory /zkl-<name>;
 * world a power of two) -- the host-side all-reduce / all-gather of per-round
 * partial sums.  zkl_sumcheck_prove_sharded is zkl_sumcheck_prove for a claim
 * whose hypercube is sharded cyclically on its low log2(world) index bits:
 * `tables` are this rank's shard (entries i*world + rank, 2^(num_vars -
 * log2 world) each), num_vars / post_add are the global claim's, and every
 * rank returns the same rounds, point, finals and end state as the unsharded
 * prover (replaces prove_sumcheck, sumcheck.py:98-130, for one shard).
 * zkl_shard_exchange: all-gather of nbytes per rank (out: world * nbytes). */
/* Exact C = A B for row-major int16 A (M x K), B (K x N) into int64 C
 * (M x N), on the tensor cores (byte-sliced mma.sync s8/u8): the wide
 * products of the LoRA-block witness (model.py:479-487 computes them with a
 * Python triple loop).  Any shape; K unbounded (int64 accumulation). */
int zkl_igemm_i16(const int16_t* A, const int16_t* B, int64_t* C, int M, int K, int N,
                  void* stream);
/* The same product through a library int8 GEMM (the tcgen05 tensor cores via
 * cuBLASLt): zkl_split_i16 writes each int16 entry's planes hi = a >> 8 and
 * lo = (a & 255) - 128 (so a = 256 hi + lo + 128); with HH = Ah Bh,
 * HL = Ah Bl, LH = Al Bh, LL = Al Bl (int32, M x N) and the row sums of A /
 * column sums of B, zkl_igemm_combine writes
 *   C = 65536 HH + 256 (HL + LH) + LL + 128 (rowA_i + colB_j) - 16384 K,
 * exact for K <= 2^16 (every int32 plane product below 2^30). */
int zkl_split_i16(const int16_t* src, uint64_t n, int8_t* hi, int8_t* lo, void* stream);
int zkl_igemm_combine(const int32_t* hh, const int32_t* hl, const int32_t* lh, const int32_t* ll,
                      const int64_t* rowA, const int64_t* colB, int64_t K, int64_t* C, int M,
                      int N, void* stream);

/* Hyrax row commitments (replaces commit.py:87-115 `commit`, the Pedersen
 * multi-exponentiation of each row, in the Schnorr groups of group.py:64-70):
 * group 0 = q = 96 p + 1 (33-byte elements; exponents BLS12-381 Fr, 8 words),
 * group 1 = q = 52 (2^61 - 1) + 1 (9-byte elements; test-field exponents, 2
 * words).  zkl_commit_tables fills a device buffer of
 * zkl_commit_table_bytes(group, ngen) bytes with fixed-base window tables for
 * ngen generators (canonical LE, element-size bytes each; the key's column
 * generators, then its blinding generator).  zkl_commit_rows: `values`
 * (device) holds rows x cols canonical exponents (little-endian 32-bit words)
 * of the table laid out row-major as split_shape(n) (commit.py:25-29);
 * `blinding` (device, rows exponents) may be NULL (binding-only mode), and
 * blind_gen is the index of the blinding generator's table; rows_out
 * (host) receives the rows' group elements, canonical LE.  Bit-identical to
 * the reference's row commitments. */
uint64_t zkl_commit_table_bytes(int group, int ngen);
int zkl_commit_tables(int group, const uint8_t* gens_canon, int ngen, void* tables, void* stream);
int zkl_commit_rows(int group, const void* tables, int cols, const void* values,
                    const void* blinding, int blind_gen, int rows, uint8_t* rows_out,
                    void* stream);

int zkl_shard_open(const char* name, int rank, int world);
int zkl_shard_close(void);
int zkl_shard_world(void);
int zkl_shard_exchange(const void* mine, uint64_t nbytes, void* out);
int zkl_sumcheck_prove_sharded(int field, void* const* tables, int k, int num_vars, int degree,
                               int nterms, const int32_t* nfactors, const int32_t* factors,
                               const uint8_t* coeffs_canon, const uint8_t* post_add_canon,
                               const uint8_t* post_mul_canon, uint8_t* state_inout,
                               uint8_t* rounds_out, uint8_t* point_out, uint8_t* finals_out,
                               void* stream);

/* Host SHAKE-256 (FIPS 202) and transcript primitives (transcript.py:13-42),
 * exported for cross-checks against hashlib; no GPU involved. */
int zkl_shake256(const uint8_t* in, uint64_t len, uint8_t* out, uint64_t outlen);
int zkl_transcript_append(uint8_t* state_inout, const uint8_t* label, uint64_t label_len,
                          const uint8_t* data, uint64_t data_len);
int zkl_transcript_challenge(int field, uint8_t* state_inout, const uint8_t* label,
                             uint64_t label_len, uint8_t* out_canon);
/* count appends of canonical little-endian integers (stride bytes each,
 * absorbed in their minimal >= 1-byte encoding) under one label: the
 * reference's per-coordinate / per-value opening records (commit.py:192-195). */
int zkl_transcript_append_ints(uint8_t* state_inout, const uint8_t* label, uint64_t label_len,
                               const uint8_t* values, uint64_t count, uint64_t stride);
/* Transcript.challenge_vector (transcript.py:44-45): count challenges under
 * "<label>/<i>", canonical scalars into out_canon.  Labels are (pointer,
 * length): any length, embedded NULs hashed as given. */
int zkl_transcript_challenge_vector(int field, uint8_t* state_inout, const uint8_t* label,
                                    uint64_t label_len, uint64_t count, uint8_t* out_canon);

/* After the last round: final_values[j] = fold(tables[j], r_last)[0]
 * (sumcheck.py:129-130), tables of size 2. */
int zkl_sumcheck_finish(int field, void* const* tables, int k, const uint8_t* r_last_canon,
                        uint8_t* finals_out_host, void* stream);

/* batch_inverse (field.py:34-46): dst[i] = 1/(src[i] + add) (add_canon may
 * be NULL).  ZKL_ERR_ZERO with *first_zero = first index whose input is 0;
 * lookup.py:163-171 uses the same check as its pole test. */
int zkl_batch_inverse(int field, void* dst, const void* src, uint64_t n, const uint8_t* add_canon,
                      int64_t* first_zero, void* stream);

/* compute_multiplicities (lookup.py:91-99): counts[j] (uint32, device) =
 * #{i : secret[i] == table[last j with that value]}; ZKL_ERR_MISSING with
 * *first_miss = first secret index not in the table. */
int zkl_multiplicities(int field, const void* secret, uint64_t d, const void* table, uint64_t n,
                       uint32_t* counts, int64_t* first_miss, void* stream);

/* zkl_multiplicities plus, per secret entry, the table index it matched
 * (index_out: d uint32 on the device; 0xffffffff where it missed).  With
 * it the lookup prover gathers 1/(beta + s_i) = 1/(beta + t_idx(i)) from
 * the table-side inversion (lookup.py:163-171) instead of inverting d
 * secret entries. */
int zkl_multiplicities_index(int field, const void* secret, uint64_t d, const void* table,
                             uint64_t n, uint32_t* counts, uint32_t* index_out,
                             int64_t* first_miss, void* stream);

/* zkl_multiplicities_index for a pair lookup (gadgets.py:679-688) whose table
 * x column is the consecutive range table_x0 .. table_x0 + n - 1
 * (tables.py:142-152): query i with 0 <= x[i] - table_x0 < n and
 * y[i] == table_y[x[i] - table_x0] is binned directly; every other query is
 * looked up by its combined value secret[i] = x[i] + alpha y[i].  x, y:
 * ZKL_MT_I16 / ZKL_MT_I32 device columns of d entries; table_y: int32, n
 * entries; table: the combined table (n field elements).  Same outputs and
 * errors as zkl_multiplicities_index (secret may be NULL: a query off its table
 * row is then reported as a miss without the hash probe, for an integer-only
 * first pass); ZKL_ERR_UNSUPPORTED (nothing written
 * but the hash slots) when the combined table has duplicate values or the
 * column types are not int16/int32. */
int zkl_pair_multiplicities(int field, const void* x, int x_type, const void* y, int y_type,
                            uint64_t d, int64_t table_x0, const int32_t* table_y,
                            const void* secret, const void* table, uint64_t n, uint32_t* counts,
                            uint32_t* index_out, int64_t* first_miss, void* stream);

/* rescale_witness (gadgets.py:563-580) / swiglu_witness narrowing: for each
 * signed wide entry w (int16 / int32 / int64 column, wide_type 1 / 2 / 3),
 * centered_divmod (quantize.py:101-104) q = floor((w + divisor/2) / divisor),
 * r = w - divisor q, written as int16 q_out[i] and r_out[i] = r * lift.  A
 * quotient outside [qmin, qmax] is the reference's RangeViolation
 * (gadgets.py:575): ZKL_ERR_MISSING with *first_bad = its first index and
 * *n_bad = the number of such entries.  Nothing is clamped. */
int zkl_rescale_witness(const void* wide, int wide_type, uint64_t n, int64_t divisor,
                        int64_t lift, int64_t qmin, int64_t qmax, int16_t* q_out, int16_t* r_out,
                        int64_t* first_bad, uint64_t* n_bad, void* stream);

/* compute_multiplicities (lookup.py:91-99) for a single-column table that is
 * the consecutive integer range table_x0 .. table_x0+n-1 (quant_range /
 * residue_range, tables.py:109-117) and a secret given as a signed int16 /
 * int32 / int64 device column (x_type 1 / 2 / 3): counts[n] (uint32), the
 * table index of every entry in index_out[d] (may be NULL), ZKL_ERR_MISSING
 * with *first_miss = the first entry outside the range.  Field-independent:
 * the secret is never lifted. */
int zkl_range_multiplicities(const void* x, int x_type, uint64_t d, int64_t table_x0,
                             uint64_t n, uint32_t* counts, uint32_t* index_out,
                             int64_t* first_miss, void* stream);

/* dst[i] = src[idx[i]] (+ add when add_canon != NULL), i < n; every idx[i]
 * must be < src_n (caller-checked).  The secret-side logUp columns
 * (lookup.py:175-202) of a lookup whose secret entries are table entries. */
int zkl_gather(int field, void* dst, const void* src, uint64_t src_n, const uint32_t* idx,
               uint64_t n, const uint8_t* add_canon, void* stream);

/* y = M x (transpose 0) or M^T x (transpose 1); M row-major rows x cols of
 * type mtype (ZKL_MT_*), x/y device field vectors.  The MLE partial
 * evaluations behind the factored zkMat prover (gadgets.py:210-251). */
int zkl_matvec(int field, int mtype, const void* M, uint64_t rows, uint64_t cols, int transpose,
               const void* x, void* y, void* stream);

/* The whole sumcheck of prove_matmul (gadgets.py:241-251) for C = A B:
 * draws r_u (d0 coordinates, labels "matmul/r_u/<i>") and r_v (d2,
 * "matmul/r_v/<i>"), absorbs the claim (sumcheck.py:90-95) and emits the
 * d0+d1+d2 rounds of the reference's replicated-table claim
 * (gadgets.py:210-251), bit-identical, without materialising the tables
 * (factored prover).  A: 2^d0 x 2^d1, B: 2^d1 x 2^d2,
 * C: 2^d0 x 2^d2, row-major device matrices of type ZKL_MT_* (integers are
 * signed, value x mod p; ZKL_MT_FIELD = storage-form elements).
 * state_inout: 64-byte transcript state (transcript.py:24-42), advanced in
 * place.  Outputs (canonical LE): rounds_out (d0+d1+d2) x 4 scalars,
 * point_out d0+d1+d2 scalars, finals_out 4 scalars (the four tables folded
 * at the point: eq, A, B, C). */
int zkl_matmul_prove(int field, int a_type, const void* A, int b_type, const void* B, int c_type,
                     const void* C, int d0, int d1, int d2, uint8_t* state_inout,
                     uint8_t* rounds_out, uint8_t* point_out, uint8_t* finals_out, void* stream);

/* zkl_matmul_prove for a sequence of claims on one transcript, with the
 * records a caller appends between claims (e.g. a gadget tag) passed in:
 * claim i is preceded by the transcript records pre[pre_off[i] ..
 * pre_off[i+1]) -- each u16le |label| || label || u64le |data| || data, the
 * framing of transcript.py:13-35 -- and then proven exactly as
 * zkl_matmul_prove would.  Same bytes as the one-claim calls in a loop
 * (gadgets.py:241-251 per claim), but the next claim's challenge draws and
 * matvecs are queued while the previous claim's last fold runs.
 * types / mats / dims: 3 entries per claim (A, B, C; d0, d1, d2).  Outputs
 * are the per-claim outputs of zkl_matmul_prove concatenated in claim order.
 * pre / pre_off may be NULL (no records). */
int zkl_matmul_prove_batch(int field, int nclaims, const int* types, const void* const* mats,
                           const int* dims, const uint8_t* pre, const uint64_t* pre_off,
                           uint8_t* state_inout, uint8_t* rounds_out, uint8_t* point_out,
                           uint8_t* finals_out, void* stream);

/* The logUp Eq.-7 sumcheck (lookup.py:188-219) for a secret larger than the
 * table (d = 2^num_vars > n = 2^tile_log, tile_log >= 5): runs the first
 * `rounds` = num_vars - tile_log rounds and appends exactly the reference's
 * transcript bytes, without materialising the replicated table side (B,
 * T+beta, M depend on index mod n; the indicator == 1) or the eq table E (it
 * is factored through the eq point u).  Afterwards A and S+beta are folded by
 * the last challenge (their first n entries hold the bound tables) and
 * tables[0] holds E bound at the point (n entries).
 * tables: E_out (n entries, written), A, S+beta (2^num_vars, consumed),
 * B, T+beta, M (n entries, read).  u_canon: the eq point (num_vars scalars);
 * coeffs: the five term coefficients (lookup.py:116-126), canonical.
 * flags bit 0: A = 1/(S+beta) entrywise (lets round 0 skip two products).
 * flags bit 1 (indexed, rounds >= 2): tables[6] is the uint32 query -> table
 * index of a lookup whose secret entries are table entries; A = B[index] and
 * S+beta = (T+beta)[index] are read through it in rounds 0 and 1 and never
 * materialised, and tables[1], tables[2] are 2^(num_vars-1)-entry outputs
 * written by the first fold.
 * The remaining tile_log rounds run through zkl_sumcheck_prove on the 7
 * tables of n entries (indicator = ones).  ZKL_ERR_UNSUPPORTED in stepwise
 * mode or for n < 32. */
int zkl_logup_tiled_rounds(int field, void* const* tables, int tile_log, int num_vars, int rounds,
                           const uint8_t* u_canon, const uint8_t* coeffs_canon, int flags,
                           uint8_t* state_inout, uint8_t* rounds_out, uint8_t* point_out,
                           void* stream);

/* CUDA-event profiler for benchmarks: when enabled, the library brackets
 * each kernel family on its launching stream.  kind 0: matrix-vector
 * products (bytes = matrix + vectors), 1: sumcheck phases (persistent round
 * engine; units = rounds), 2: eq tables.  zkl_prof_collect synchronises on
 * the recorded events and returns total milliseconds, algorithmic bytes,
 * units and launch groups of one kind since the last collect. */
int zkl_prof_enable(int on);
int zkl_prof_collect(int kind, double* ms, double* bytes, double* units, uint64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* ZKL_B200_H */
