"""zkMat sumcheck: reference replicated claim and the factored restatement.

Reference: /root/reference/pkg/src/zklora/gadgets.py:210-251.  The sumcheck
boundary used throughout this repo starts at the r_u / r_v draws
(gadgets.py:241-242) and ends when prove_sumcheck returns (gadgets.py:251);
operand absorption (gadgets.py:240) and openings (gadgets.py:254-265) sit
outside it.

``prove_dense`` materialises the four replicated tables exactly as the
reference does (O(2^(d0+d1+d2)) memory; small shapes only).
``prove_factored`` produces bit-identical rounds / point / final values from
MLE partial evaluations and three short two-factor sumchecks (derivation in
DESIGN.md).  It is the large-shape oracle; it is
pinned against ``prove_dense`` and the reference goldens at small shapes.

Matrices are given as row-major Python int lists (field residues or signed
ints) or numpy integer arrays (|entry| < 2^47) for the large-shape path.
"""

import numpy as np

from .multilinear import eq_vec, fold_msb
from .prime import inv
from .sc import absorb_claim, prove as sc_prove


def matmul_terms(d1, p):
    """gadgets.py:246: [eq*A*B, -2^-d1 * eq*C]."""
    return [(1, (0, 1, 2)), ((-inv(1 << d1, p)) % p, (0, 3))]


def replicated_tables(A, B, C, eu, ev, d0, d1, d2, p):
    """gadgets.py:210-227, index = u|w|v (u most significant)."""
    D0, D1, D2 = 1 << d0, 1 << d1, 1 << d2
    t_eq, t_a, t_b, t_c = [], [], [], []
    for u in range(D0):
        for w in range(D1):
            av = A[u * D1 + w]
            for v in range(D2):
                t_eq.append(eu[u] * ev[v] % p)
                t_a.append(av)
                t_b.append(B[w * D2 + v])
                t_c.append(C[u * D2 + v])
    return [t_eq, t_a, t_b, t_c]


def prove_dense(A, B, C, dims, tr):
    """Reference algorithm: gadgets.py:241-251 then sumcheck.py:98-130."""
    d0, d1, d2 = dims
    p = tr.modulus
    r_u = tr.challenge_vector(b"matmul/r_u", d0)
    r_v = tr.challenge_vector(b"matmul/r_v", d2)
    tabs = replicated_tables(A, B, C, eq_vec(r_u, p), eq_vec(r_v, p), d0, d1, d2, p)
    return sc_prove(0, tabs, matmul_terms(d1, p), 3, tr)


# ---------------------------------------------------------------------------
# exact integer-matrix x field-vector products (numpy, float64-exact limbs)


def _limbs16(vec):
    """Field vector -> (16, n) float64 array of 16-bit limbs."""
    n = len(vec)
    raw = b"".join(int(v).to_bytes(32, "little") for v in vec)
    arr = np.frombuffer(raw, dtype="<u2").reshape(n, 16).T
    return arr.astype(np.float64)


def _split_matrix(M):
    """Signed int64 matrix -> list of (shift, float64 limb matrix), exact."""
    M = np.asarray(M, dtype=np.int64)
    if np.abs(M).max(initial=0) < (1 << 15):
        return [(0, M.astype(np.float64))]
    lo = (M & 0xFFFF).astype(np.float64)
    mid = ((M >> 16) & 0xFFFF).astype(np.float64)
    hi = M >> 32
    assert np.abs(hi).max(initial=0) < (1 << 15), "entries must be < 2^47"
    return [(0, lo), (16, mid), (32, hi.astype(np.float64))]


def int_matvec(M, vec, p):
    """(M @ vec) mod p for a signed integer matrix M (rows x cols)."""
    V = _limbs16(vec)  # (16, cols)
    acc = [0] * M.shape[0]
    for shift, part in _split_matrix(M):
        prod = part @ V.T  # (rows, 16), every entry an exact integer < 2^53
        prod = np.rint(prod).astype(np.int64)
        for k in range(16):
            col = prod[:, k].tolist()
            sh = shift + 16 * k
            for r, x in enumerate(col):
                acc[r] += x << sh
    return [a % p for a in acc]


def _matvec(M, vec, p, D_rows, D_cols):
    if isinstance(M, np.ndarray):
        return int_matvec(M.reshape(D_rows, D_cols), vec, p)
    out = []
    for r in range(D_rows):
        base = r * D_cols
        s = 0
        for c in range(D_cols):
            s += M[base + c] * vec[c]
        out.append(s % p)
    return out


def _vecmat(vec, M, p, D_rows, D_cols):
    if isinstance(M, np.ndarray):
        return int_matvec(M.reshape(D_rows, D_cols).T, vec, p)
    out = [0] * D_cols
    for r in range(D_rows):
        w = vec[r]
        base = r * D_cols
        for c in range(D_cols):
            out[c] += w * M[base + c]
    return [o % p for o in out]


def _two_factor_round(f, g, p):
    """sum_i f_x g_x at x = 0..3 over the MSB pairs of two tables."""
    h = len(f) >> 1
    ev = [0, 0, 0, 0]
    for i in range(h):
        f0, f1 = f[i], f[i + h]
        g0, g1 = g[i], g[i + h]
        df, dg = f1 - f0, g1 - g0
        ev[0] += f0 * g0
        ev[1] += f1 * g1
        ev[2] += (f1 + df) * (g1 + dg)
        ev[3] += (f1 + 2 * df) * (g1 + 2 * dg)
    return [e % p for e in ev]


def _emit(tr, ev):
    for e in ev:
        tr.append(b"sumcheck/eval", e)
    return tr.challenge(b"sumcheck/round")


def prove_factored(A, B, C, dims, tr):
    """Bit-identical to prove_dense without materialising 2^(d0+d1+d2) tables."""
    d0, d1, d2 = dims
    D0, D1, D2 = 1 << d0, 1 << d1, 1 << d2
    p = tr.modulus
    r_u = tr.challenge_vector(b"matmul/r_u", d0)
    r_v = tr.challenge_vector(b"matmul/r_v", d2)
    terms = matmul_terms(d1, p)
    cneg = terms[1][0]
    absorb_claim(tr, 0, terms, 3, d0 + d1 + d2)
    E_u, E_v = eq_vec(r_u, p), eq_vec(r_v, p)
    rounds, point = [], []

    # U phase: sum_u E_u(u) h(u), h = A (B E_v) + c 2^d1 (C E_v)
    bv = _matvec(B, E_v, p, D1, D2)
    cv = _matvec(C, E_v, p, D0, D2)
    abv = _matvec(A, bv, p, D0, D1)
    k = cneg * pow(2, d1, p) % p
    f, g = E_u, [(x + k * y) % p for x, y in zip(abv, cv)]
    for _ in range(d0):
        ev = _two_factor_round(f, g, p)
        rounds.append(tuple(ev))
        r = _emit(tr, ev)
        point.append(r)
        f, g = fold_msb(f, r, p), fold_msb(g, r, p)
    e_hat = f[0]
    E_ru = eq_vec(point[:d0], p)

    # W phase: E_hat * [sum_w a(w) bv(w) + c 2^(rem) kappa]
    a = _vecmat(E_ru, A, p, D0, D1)
    cu = _vecmat(E_ru, C, p, D0, D2)
    kappa = sum(x * y for x, y in zip(cu, E_v)) % p
    f, g = a, bv
    for j in range(d1):
        ev = _two_factor_round(f, g, p)
        const = cneg * pow(2, d1 - j - 1, p) % p * kappa % p
        ev = [e_hat * ((e + const) % p) % p for e in ev]
        rounds.append(tuple(ev))
        r = _emit(tr, ev)
        point.append(r)
        f, g = fold_msb(f, r, p), fold_msb(g, r, p)
    alpha_s = f[0]
    E_rw = eq_vec(point[d0 : d0 + d1], p)

    # V phase: E_hat * sum_v E_v(v) [alpha_s bw(v) + c cu(v)]
    bw = _vecmat(E_rw, B, p, D1, D2)
    f = E_v
    g = [(alpha_s * x + cneg * y) % p for x, y in zip(bw, cu)]
    t_b, t_c = bw, cu
    for _ in range(d2):
        ev = _two_factor_round(f, g, p)
        ev = [e_hat * e % p for e in ev]
        rounds.append(tuple(ev))
        r = _emit(tr, ev)
        point.append(r)
        f, g = fold_msb(f, r, p), fold_msb(g, r, p)
        t_b, t_c = fold_msb(t_b, r, p), fold_msb(t_c, r, p)
    finals = (e_hat * f[0] % p, alpha_s, t_b[0], t_c[0])
    return rounds, finals, point


def mle_matrix(M, rows_pt, cols_pt, p):
    """MLE of a row-major matrix at (row point || col point)."""
    Dr, Dc = 1 << len(rows_pt), 1 << len(cols_pt)
    col = _matvec(M, eq_vec(cols_pt, p), p, Dr, Dc)
    er = eq_vec(rows_pt, p)
    return sum(x * y for x, y in zip(er, col)) % p
