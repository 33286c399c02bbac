/* CPU oracle kernels for large-size parity (TEST INFRASTRUCTURE ONLY).
 *
 * Plain C (gcc -O3 -fopenmp) restatement of the reference's field and MLE
 * arithmetic so the oracle can check the GPU path at BASELINE sizes
 * (2^21 - 2^25 entries) where the pure-Python oracle would take hours:
 *
 *   field  /root/reference/pkg/src/zklora/field.py:9-46   (BLS12-381 Fr and
 *          2^61-1; inverse, Montgomery-trick batch_inverse)
 *   mle    mle.py:50-82   (MSB-first fold_table, eq_table)
 *   round  sumcheck.py:110-123 (evaluations at x = 0..degree of
 *          sum_i sum_t c_t prod_{f in t} table_f(x, i), every one computed
 *          from the tables, g(1) included)
 *
 * Only the oracle Python modules drive it (oracle/fast.py, ctypes); the transcript stays
 * in Python (oracle/fs.py, hashlib).  Fr elements are 4 x 64-bit limbs in
 * Montgomery form (R = 2^256, CIOS with unsigned __int128); 2^61-1 elements
 * are canonical uint64.  Scalars cross the ABI as 32-byte canonical little
 * endian.  fid 0 = Fr, 1 = 2^61-1 (the GPU library's numbering).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- Fr */
static const uint64_t P[4] = {0xffffffff00000001ull, 0x53bda402fffe5bfeull,
                              0x3339d80809a1d805ull, 0x73eda753299d7d48ull};
static const uint64_t R2[4] = {0xc999e990f3f29c6dull, 0x2b6cedcb87925c23ull,
                               0x05d314967254398full, 0x0748d9d99f59ff11ull};
static const uint64_t NINV = 0xfffffffeffffffffull; /* -p^-1 mod 2^64 */

static inline int geq_p(const uint64_t a[4]) {
  for (int i = 3; i >= 0; i--) {
    if (a[i] > P[i]) return 1;
    if (a[i] < P[i]) return 0;
  }
  return 1;
}

static inline void sub_p(uint64_t a[4]) {
  u128 br = 0;
  for (int i = 0; i < 4; i++) {
    u128 d = (u128)a[i] - P[i] - br;
    a[i] = (uint64_t)d;
    br = (d >> 64) & 1;
  }
}

static inline void fr_add(uint64_t r[4], const uint64_t a[4], const uint64_t b[4]) {
  u128 c = 0;
  for (int i = 0; i < 4; i++) {
    c += (u128)a[i] + b[i];
    r[i] = (uint64_t)c;
    c >>= 64;
  }
  if (c || geq_p(r)) sub_p(r); /* p < 2^255: a + b < 2^256, c is always 0 */
}

static inline void fr_sub(uint64_t r[4], const uint64_t a[4], const uint64_t b[4]) {
  u128 br = 0;
  uint64_t t[4];
  for (int i = 0; i < 4; i++) {
    u128 d = (u128)a[i] - b[i] - br;
    t[i] = (uint64_t)d;
    br = (d >> 64) & 1;
  }
  if (br) {
    u128 c = 0;
    for (int i = 0; i < 4; i++) {
      c += (u128)t[i] + P[i];
      t[i] = (uint64_t)c;
      c >>= 64;
    }
  }
  memcpy(r, t, 32);
}

/* CIOS Montgomery product a*b*R^-1 mod p */
static inline void fr_mul(uint64_t r[4], const uint64_t a[4], const uint64_t b[4]) {
  uint64_t t[6] = {0, 0, 0, 0, 0, 0};
  for (int i = 0; i < 4; i++) {
    u128 c = 0;
    for (int j = 0; j < 4; j++) {
      c += (u128)a[j] * b[i] + t[j];
      t[j] = (uint64_t)c;
      c >>= 64;
    }
    c += t[4];
    t[4] = (uint64_t)c;
    t[5] = (uint64_t)(c >> 64);
    uint64_t m = t[0] * NINV;
    c = (u128)m * P[0] + t[0];
    c >>= 64;
    for (int j = 1; j < 4; j++) {
      c += (u128)m * P[j] + t[j];
      t[j - 1] = (uint64_t)c;
      c >>= 64;
    }
    c += t[4];
    t[3] = (uint64_t)c;
    t[4] = t[5] + (uint64_t)(c >> 64);
  }
  memcpy(r, t, 32);
  if (t[4] || geq_p(r)) sub_p(r);
}

static void fr_from_canon(uint64_t r[4], const uint8_t b[32]) {
  uint64_t a[4];
  memcpy(a, b, 32);
  while (geq_p(a)) sub_p(a);
  fr_mul(r, a, R2);
}

static void fr_to_canon(uint8_t b[32], const uint64_t a[4]) {
  static const uint64_t one[4] = {1, 0, 0, 0};
  uint64_t r[4];
  fr_mul(r, a, one);
  memcpy(b, r, 32);
}

/* ---------------------------------------------------------------- M61 */
static const uint64_t M61 = (1ull << 61) - 1;

static inline uint64_t m61_red(u128 x) {
  uint64_t lo = (uint64_t)(x & M61), hi = (uint64_t)(x >> 61);
  uint64_t s = lo + hi;
  s = (s & M61) + (s >> 61);
  return s >= M61 ? s - M61 : s;
}
static inline uint64_t m61_add(uint64_t a, uint64_t b) {
  uint64_t s = a + b;
  return s >= M61 ? s - M61 : s;
}
static inline uint64_t m61_sub(uint64_t a, uint64_t b) { return a >= b ? a - b : a + M61 - b; }
static inline uint64_t m61_mul(uint64_t a, uint64_t b) { return m61_red((u128)a * b); }

/* ------------------------------------------------- generic element ops */
/* W = words per element: 4 (Fr, Montgomery) or 1 (M61, canonical) */
#define WORDS(fid) ((fid) == 0 ? 4 : 1)

static inline void e_add(int fid, uint64_t* r, const uint64_t* a, const uint64_t* b) {
  if (fid == 0) fr_add(r, a, b);
  else r[0] = m61_add(a[0], b[0]);
}
static inline void e_sub(int fid, uint64_t* r, const uint64_t* a, const uint64_t* b) {
  if (fid == 0) fr_sub(r, a, b);
  else r[0] = m61_sub(a[0], b[0]);
}
static inline void e_mul(int fid, uint64_t* r, const uint64_t* a, const uint64_t* b) {
  if (fid == 0) fr_mul(r, a, b);
  else r[0] = m61_mul(a[0], b[0]);
}
static void e_from_canon(int fid, uint64_t* r, const uint8_t* b) {
  if (fid == 0) {
    fr_from_canon(r, b);
  } else {
    uint64_t v;
    memcpy(&v, b, 8); /* callers pass values already reduced mod p */
    r[0] = v % M61;
  }
}
static void e_to_canon(int fid, uint8_t* b, const uint64_t* a) {
  if (fid == 0) {
    fr_to_canon(b, a);
  } else {
    memset(b, 0, 32);
    memcpy(b, a, 8);
  }
}

static void e_from_i64(int fid, uint64_t* r, int64_t v) {
  uint8_t b[32];
  memset(b, 0, 32);
  if (fid == 0) {
    /* v mod p as canonical bytes: negative v -> p - |v| (field.py:54-55) */
    uint64_t a[4] = {v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v, 0, 0, 0};
    if (v < 0) {
      uint64_t t[4];
      memcpy(t, P, 32);
      u128 br = 0;
      for (int i = 0; i < 4; i++) {
        u128 d = (u128)t[i] - a[i] - br;
        t[i] = (uint64_t)d;
        br = (d >> 64) & 1;
      }
      memcpy(b, t, 32);
    } else {
      memcpy(b, a, 32);
    }
    fr_from_canon(r, b);
  } else {
    r[0] = v < 0 ? M61 - ((uint64_t)(-(v + 1)) + 1) % M61 : (uint64_t)v % M61;
    if (r[0] == M61) r[0] = 0;
  }
}

/* ------------------------------------------------------------- exports */
int or_words(int fid) { return WORDS(fid); }

void or_from_canon(int fid, const uint8_t* bytes, uint64_t n, uint64_t* out) {
  const int W = WORDS(fid);
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; i++) e_from_canon(fid, out + i * W, bytes + 32 * i);
}

void or_to_canon(int fid, const uint64_t* in, uint64_t n, uint8_t* bytes) {
  const int W = WORDS(fid);
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; i++) e_to_canon(fid, bytes + 32 * i, in + i * W);
}

/* signed int64 column -> field (x mod p) */
void or_from_i64(int fid, const int64_t* x, uint64_t n, uint64_t* out) {
  const int W = WORDS(fid);
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; i++) e_from_i64(fid, out + i * W, x[i]);
}

/* out[i] = x[i] + alpha * y[i]  (tables.py:131-140 for signed int columns) */
void or_pair_combine(int fid, const int64_t* x, const int64_t* y, uint64_t n,
                     const uint8_t* alpha, uint64_t* out) {
  const int W = WORDS(fid);
  uint64_t a[4];
  e_from_canon(fid, a, alpha);
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; i++) {
    uint64_t xv[4], yv[4];
    e_from_i64(fid, xv, x[i]);
    e_from_i64(fid, yv, y[i]);
    e_mul(fid, yv, yv, a);
    e_add(fid, out + i * W, xv, yv);
  }
}

/* out[i] = a[i] * b[i] */
void or_mul(int fid, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t* out) {
  const int W = WORDS(fid);
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; i++) e_mul(fid, out + i * W, a + i * W, b + i * W);
}

/* t[i] += c */
void or_add_const(int fid, uint64_t* t, uint64_t n, const uint8_t* c) {
  const int W = WORDS(fid);
  uint64_t cv[4];
  e_from_canon(fid, cv, c);
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; i++) e_add(fid, t + i * W, t + i * W, cv);
}

/* eq(point, .) over {0,1}^m, point[0] paired with the MSB (mle.py:67-82) */
void or_eq_table(int fid, const uint8_t* point, int m, uint64_t* out) {
  const int W = WORDS(fid);
  uint64_t one[4];
  e_from_i64(fid, one, 1);
  memcpy(out, one, 8 * W);
  uint64_t size = 1;
  for (int j = 0; j < m; j++) {
    uint64_t r[4], s[4];
    e_from_canon(fid, r, point + 32 * j);
    e_sub(fid, s, one, r);
    /* entry v at index i becomes (v s) at 2i and (v r) at 2i+1 */
    uint64_t* tmp = (uint64_t*)malloc(8 * W * size);
    memcpy(tmp, out, 8 * W * size);
#pragma omp parallel for schedule(static)
    for (uint64_t i = 0; i < size; i++) {
      e_mul(fid, out + (2 * i) * W, tmp + i * W, s);
      e_mul(fid, out + (2 * i + 1) * W, tmp + i * W, r);
    }
    free(tmp);
    size <<= 1;
  }
}

/* Montgomery-trick batch inversion of (in[i] + add); returns the first index
 * whose input is zero (field.py:38-39), else -1.  Chunked: per-chunk prefix
 * products, one inversion per chunk (Fermat), back-substitution. */
static void e_pow(int fid, uint64_t* r, const uint64_t* a, const uint64_t* e4) {
  uint64_t acc[4], b[4];
  e_from_i64(fid, acc, 1);
  memcpy(b, a, 32);
  for (int w = 0; w < 4; w++)
    for (int bit = 0; bit < 64; bit++) {
      if ((e4[w] >> bit) & 1) e_mul(fid, acc, acc, b);
      e_mul(fid, b, b, b);
    }
  memcpy(r, acc, 32);
}

static void e_inv(int fid, uint64_t* r, const uint64_t* a) {
  uint64_t e[4];
  if (fid == 0) {
    memcpy(e, P, 32);
    e[0] -= 2;
  } else {
    e[0] = M61 - 2;
    e[1] = e[2] = e[3] = 0;
  }
  e_pow(fid, r, a, e);
}

static int e_is_zero(int fid, const uint64_t* a) {
  if (fid == 0) return (a[0] | a[1] | a[2] | a[3]) == 0;
  return a[0] == 0;
}

int64_t or_batch_inverse(int fid, const uint64_t* in, uint64_t n, const uint8_t* add,
                         uint64_t* out) {
  const int W = WORDS(fid);
  uint64_t av[4] = {0, 0, 0, 0};
  if (add) e_from_canon(fid, av, add);
  int64_t first_zero = -1;
  const uint64_t CH = 4096;
  const uint64_t nch = (n + CH - 1) / CH;
#pragma omp parallel for schedule(dynamic, 4)
  for (uint64_t c = 0; c < nch; c++) {
    const uint64_t lo = c * CH, hi = lo + CH < n ? lo + CH : n;
    uint64_t acc[4];
    e_from_i64(fid, acc, 1);
    int zero = 0;
    for (uint64_t i = lo; i < hi; i++) { /* out[i] = prefix product before i */
      uint64_t x[4];
      e_add(fid, x, in + i * W, av);
      if (e_is_zero(fid, x)) {
        zero = 1;
#pragma omp critical
        if (first_zero < 0 || (int64_t)i < first_zero) first_zero = (int64_t)i;
        break;
      }
      memcpy(out + i * W, acc, 8 * W);
      e_mul(fid, acc, acc, x);
    }
    if (zero) continue;
    uint64_t inv[4];
    e_inv(fid, inv, acc);
    for (uint64_t i = hi; i-- > lo;) {
      uint64_t x[4], t[4];
      e_add(fid, x, in + i * W, av);
      e_mul(fid, t, out + i * W, inv); /* 1/x_i */
      e_mul(fid, inv, inv, x);
      memcpy(out + i * W, t, 8 * W);
    }
  }
  return first_zero;
}

/* One sumcheck round (sumcheck.py:110-123): evals[x] for x = 0..degree of
 * sum over the pairs (i, i + half) of sum_t coeff_t prod_{f in factors_t}
 * table_f(x), table_f(x) = lo + x (hi - lo).  terms are given as
 * (coefficient, factor list) flattened: fac[off[t] .. off[t+1]). */
void or_round(int fid, uint64_t* const* tables, int k, uint64_t half, const int* fac,
              const int* off, const uint8_t* coeffs, int nterms, int degree,
              uint8_t* evals_out) {
  const int W = WORDS(fid);
  uint64_t cf[16][4];
  for (int t = 0; t < nterms; t++) e_from_canon(fid, cf[t], coeffs + 32 * t);
  uint64_t one[4];
  e_from_i64(fid, one, 1);
  uint64_t total[4][16][4]; /* per x, per term raw sums (coefficients at the end) */
  memset(total, 0, sizeof total);
#pragma omp parallel
  {
    uint64_t acc[4][16][4];
    memset(acc, 0, sizeof acc);
#pragma omp for schedule(static)
    for (uint64_t i = 0; i < half; i++) {
      uint64_t val[16][4], dif[16][4];
      for (int f = 0; f < k; f++) {
        memcpy(val[f], tables[f] + i * W, 8 * W);
        e_sub(fid, dif[f], tables[f] + (i + half) * W, val[f]);
      }
      for (int x = 0; x <= degree; x++) {
        if (x > 0)
          for (int f = 0; f < k; f++) e_add(fid, val[f], val[f], dif[f]);
        for (int t = 0; t < nterms; t++) {
          uint64_t prod[4];
          if (off[t] == off[t + 1]) { /* a term with no factors is the constant 1 */
            memcpy(prod, one, 8 * W);
          } else {
            memcpy(prod, val[fac[off[t]]], 8 * W);
            for (int q = off[t] + 1; q < off[t + 1]; q++) e_mul(fid, prod, prod, val[fac[q]]);
          }
          e_add(fid, acc[x][t], acc[x][t], prod);
        }
      }
    }
#pragma omp critical
    for (int x = 0; x <= degree; x++)
      for (int t = 0; t < nterms; t++) e_add(fid, total[x][t], total[x][t], acc[x][t]);
  }
  for (int x = 0; x <= degree; x++) {
    uint64_t s[4] = {0, 0, 0, 0};
    for (int t = 0; t < nterms; t++) {
      uint64_t v[4];
      e_mul(fid, v, total[x][t], cf[t]);
      e_add(fid, s, s, v);
    }
    e_to_canon(fid, evals_out + 32 * x, s);
  }
}

/* fold every table in place by r (mle.py:50-56): t[i] = t[i] + r (t[i+h] - t[i]) */
void or_fold(int fid, uint64_t* const* tables, int k, uint64_t half, const uint8_t* rb) {
  const int W = WORDS(fid);
  uint64_t r[4];
  e_from_canon(fid, r, rb);
  for (int f = 0; f < k; f++) {
    uint64_t* t = tables[f];
#pragma omp parallel for schedule(static)
    for (uint64_t i = 0; i < half; i++) {
      uint64_t d[4];
      e_sub(fid, d, t + (i + half) * W, t + i * W);
      e_mul(fid, d, d, r);
      e_add(fid, t + i * W, t + i * W, d);
    }
  }
}

/* sum_i a[i] b[i] (b NULL: sum_i a[i]) */
void or_dot(int fid, const uint64_t* a, const uint64_t* b, uint64_t n, uint8_t* out) {
  const int W = WORDS(fid);
  uint64_t tot[4] = {0, 0, 0, 0};
#pragma omp parallel
  {
    uint64_t acc[4] = {0, 0, 0, 0};
#pragma omp for schedule(static)
    for (uint64_t i = 0; i < n; i++) {
      uint64_t v[4];
      if (b) e_mul(fid, v, a + i * W, b + i * W);
      else memcpy(v, a + i * W, 8 * W);
      e_add(fid, acc, acc, v);
    }
#pragma omp critical
    e_add(fid, tot, tot, acc);
  }
  e_to_canon(fid, out, tot);
}
