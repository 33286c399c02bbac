"""Large-size oracle: the reference's dense sumcheck and logUp provers with the
per-entry arithmetic in plain C (oracle/csrc/frc.c, OpenMP) and the
transcript in Python (oracle/fs.py, hashlib).  TEST INFRASTRUCTURE ONLY.

  prove_dense   sumcheck.py:98-130  (claim absorption, per round evals at
                x = 0..degree all computed from the tables, challenge, fold)
  prove_logup   lookup.py:143-251   (multiplicities, beta with pole retries,
                batch inversions, the 7-table Eq.-7 claim, openings), for
                secrets and tables given as signed integer columns or integer
                pair columns (x + alpha y, gadgets.py:659-688)
  mle           mle.py:59-64

It is the same algorithm as oracle/sc.py and oracle/logup.py (pinned against
the reference's goldens); tests/test_oracle_golden.py checks the two agree
entry for entry at small sizes, so the C arithmetic inherits that pin.
Tables are numpy uint64 arrays of shape (n, W): W = 4 Montgomery limbs for
BLS12-381 Fr, W = 1 canonical word for 2^61-1.
"""

import ctypes
import os

import numpy as np

from .logup import MAX_RETRIES, Pole, logup_terms
from .prime import P_BIG, P_TEST, inv
from .sc import absorb_claim
from .stubcommit import stub_bytes

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libfrc.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            import subprocess

            subprocess.run(["make", "-s", "-C", HERE], check=True)
        L = ctypes.CDLL(LIB)
        vp, u64, i32, cp = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_char_p
        L.or_words.argtypes = [i32]
        L.or_from_canon.argtypes = [i32, cp, u64, vp]
        L.or_to_canon.argtypes = [i32, vp, u64, vp]
        L.or_from_i64.argtypes = [i32, vp, u64, vp]
        L.or_pair_combine.argtypes = [i32, vp, vp, u64, cp, vp]
        L.or_add_const.argtypes = [i32, vp, u64, cp]
        L.or_mul.argtypes = [i32, vp, vp, u64, vp]
        L.or_eq_table.argtypes = [i32, cp, i32, vp]
        L.or_batch_inverse.argtypes = [i32, vp, u64, cp, vp]
        L.or_batch_inverse.restype = ctypes.c_int64
        L.or_round.argtypes = [i32, vp, i32, u64, vp, vp, cp, i32, i32, vp]
        L.or_fold.argtypes = [i32, vp, i32, u64, cp]
        L.or_dot.argtypes = [i32, vp, vp, u64, vp]
        _lib = L
    return _lib


def fid_of(p):
    if p == P_BIG:
        return 0
    if p == P_TEST:
        return 1
    raise ValueError("oracle C kernels implement the reference's two fields only")


def _b(v):
    return (int(v)).to_bytes(32, "little")


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


class Field:
    def __init__(self, p):
        self.p, self.fid = p, fid_of(p)
        self.W = lib().or_words(self.fid)

    def empty(self, n):
        return np.zeros((n, self.W), dtype=np.uint64)

    def from_ints(self, x):
        x = np.ascontiguousarray(np.asarray(x, dtype=np.int64).reshape(-1))
        out = self.empty(x.size)
        lib().or_from_i64(self.fid, _ptr(x), x.size, _ptr(out))
        return out

    def from_residues(self, vals):
        vals = [int(v) % self.p for v in vals]
        raw = b"".join(_b(v) for v in vals)
        out = self.empty(len(vals))
        lib().or_from_canon(self.fid, raw, len(vals), _ptr(out))
        return out

    def to_residues(self, a):
        n = a.shape[0]
        raw = ctypes.create_string_buffer(32 * n)
        lib().or_to_canon(self.fid, _ptr(a), n, raw)
        mv = raw.raw
        return [int.from_bytes(mv[32 * i:32 * i + 32], "little") for i in range(n)]

    def scalar(self, a, i=0):
        return self.to_residues(a[i:i + 1])[0]

    def pair_combine(self, x, y, alpha):
        x = np.ascontiguousarray(np.asarray(x, dtype=np.int64).reshape(-1))
        y = np.ascontiguousarray(np.asarray(y, dtype=np.int64).reshape(-1))
        out = self.empty(x.size)
        lib().or_pair_combine(self.fid, _ptr(x), _ptr(y), x.size, _b(alpha % self.p), _ptr(out))
        return out

    def mul(self, a, b):
        out = self.empty(a.shape[0])
        lib().or_mul(self.fid, _ptr(a), _ptr(b), a.shape[0], _ptr(out))
        return out

    def add_const(self, a, c):
        a = a.copy()
        lib().or_add_const(self.fid, _ptr(a), a.shape[0], _b(c % self.p))
        return a

    def eq_table(self, point):
        out = self.empty(1 << len(point))
        lib().or_eq_table(self.fid, b"".join(_b(r % self.p) for r in point), len(point),
                          _ptr(out))
        return out

    def batch_inverse(self, a, add=None):
        """(1/(a + add), first zero index or None)."""
        out = self.empty(a.shape[0])
        z = lib().or_batch_inverse(self.fid, _ptr(a), a.shape[0],
                                   None if add is None else _b(add % self.p), _ptr(out))
        return out, (None if z < 0 else int(z))

    def dot(self, a, b=None):
        raw = ctypes.create_string_buffer(32)
        lib().or_dot(self.fid, _ptr(a), None if b is None else _ptr(b), a.shape[0], raw)
        return int.from_bytes(raw.raw, "little")

    def mle(self, a, point):
        """mle.py:59-64 by folds (a is not modified)."""
        t = a.copy()
        for r in point:
            self.fold([t], r)
            t = t[: t.shape[0] // 2]
        return self.scalar(t)

    # --- sumcheck primitives -------------------------------------------------
    def round(self, tables, terms, degree):
        half = tables[0].shape[0] // 2
        ptrs = (ctypes.c_void_p * len(tables))(*[t.ctypes.data for t in tables])
        fac, off = [], [0]
        for _, f in terms:
            fac.extend(f)
            off.append(len(fac))
        fac_a = (ctypes.c_int * max(len(fac), 1))(*fac)
        off_a = (ctypes.c_int * len(off))(*off)
        coeffs = b"".join(_b(c % self.p) for c, _ in terms)
        raw = ctypes.create_string_buffer(32 * (degree + 1))
        lib().or_round(self.fid, ptrs, len(tables), half, fac_a, off_a, coeffs, len(terms),
                       degree, raw)
        return [int.from_bytes(raw.raw[32 * x:32 * x + 32], "little") for x in range(degree + 1)]

    def fold(self, tables, r):
        """In place on each table's first half (callers slice afterwards)."""
        half = tables[0].shape[0] // 2
        ptrs = (ctypes.c_void_p * len(tables))(*[t.ctypes.data for t in tables])
        lib().or_fold(self.fid, ptrs, len(tables), half, _b(r % self.p))


def prove_dense(claimed_sum, tables, terms, degree, tr):
    """sumcheck.py:98-130 over numpy field tables (consumed): returns
    (rounds, final_values, point) like oracle.sc.prove."""
    F = Field(tr.modulus)
    cur = [np.ascontiguousarray(t) for t in tables]
    n = (cur[0].shape[0] - 1).bit_length()
    absorb_claim(tr, claimed_sum, terms, degree, n)
    rounds, point = [], []
    for _ in range(n):
        ev = F.round(cur, terms, degree)
        rounds.append(tuple(ev))
        for e in ev:
            tr.append(b"sumcheck/eval", e)
        r = tr.challenge(b"sumcheck/round")
        point.append(r)
        F.fold(cur, r)
        cur = [np.ascontiguousarray(t[: t.shape[0] // 2]) for t in cur]
    return rounds, tuple(F.scalar(t) for t in cur), point


def multiplicities_int(secret_int, table_int):
    """lookup.py:91-99 for an integer secret against a table of distinct
    integers (range / pair-table x columns): (counts, first miss or None)."""
    secret_int = np.asarray(secret_int, dtype=np.int64).reshape(-1)
    table_int = np.asarray(table_int, dtype=np.int64).reshape(-1)
    order = np.argsort(table_int, kind="stable")
    st = table_int[order]
    pos = np.searchsorted(st, secret_int, side="right") - 1
    pos = np.clip(pos, 0, len(st) - 1)
    hit = st[pos] == secret_int
    if not hit.all():
        return None, int(np.argmin(hit))
    idx = order[pos]
    return np.bincount(idx, minlength=len(table_int)).astype(np.int64), None


def _open(values, point, tr):
    """The stub opening's transcript traffic (oracle/stubcommit.py)."""
    for r in point:
        tr.append(b"open/point", r)
    for y in values:
        tr.append(b"open/value", y)


def prove_logup(F, s_field, t_field, mult, table_com, secret_com, tr):
    """lookup.py:143-251 (prove_lookup) over numpy field columns: the secret
    s (d entries) and table t (n entries) already as field elements, `mult`
    an int64 count vector; stub commitments (oracle/stubcommit.py).  Returns
    the same keys as oracle.logup.prove."""
    p = tr.modulus
    d, n = s_field.shape[0], t_field.shape[0]
    m_field = F.from_ints(mult)
    m_com = stub_bytes((n - 1).bit_length())
    tr.append(b"lookup/table", table_com)
    tr.append(b"lookup/secret", secret_com)
    tr.append(b"lookup/mult", m_com)
    retries = 0
    beta = tr.challenge(b"lookup/beta")
    while True:
        inv_s, z1 = F.batch_inverse(s_field, beta)
        inv_t, z2 = F.batch_inverse(t_field, beta)
        if z1 is None and z2 is None:
            break
        retries += 1
        if retries > MAX_RETRIES:
            raise Pole("challenge hit a pole %d times" % retries)
        tr.append(b"lookup/beta-retry", retries)
        beta = tr.challenge(b"lookup/beta")
    tr.append(b"lookup/inv-secret", stub_bytes((d - 1).bit_length()))
    tr.append(b"lookup/inv-table", stub_bytes((n - 1).bit_length()))
    alpha = tr.challenge(b"lookup/alpha")
    big = max(d, n)
    nv = (big - 1).bit_length()
    u = tr.challenge_vector(b"lookup/u", nv)
    ratio = inv(big // n, p)
    terms = logup_terms(alpha, ratio, p)
    one = F.from_ints([1])
    if d <= n:
        pad = n - d
        zpad = F.empty(pad)
        A = np.concatenate([inv_s, zpad])
        Sb = F.add_const(np.concatenate([s_field, zpad]), beta)
        ind = np.concatenate([np.repeat(one, d, axis=0), zpad])
        B, Tb, M = inv_t.copy(), F.add_const(t_field, beta), m_field.copy()
    else:
        c = d // n
        A, ind = inv_s.copy(), np.repeat(one, d, axis=0)
        Sb = F.add_const(s_field, beta)
        B, Tb, M = np.tile(inv_t, (c, 1)), np.tile(F.add_const(t_field, beta), (c, 1)), \
            np.tile(m_field, (c, 1))
    tables = [F.eq_table(u), A, Sb, ind, B, Tb, M]
    rounds, finals, point = prove_dense(alpha * alpha % p, tables, terms, 3, tr)
    d_vars, n_vars = (d - 1).bit_length(), (n - 1).bit_length()
    sp, tp = point[nv - d_vars:], point[nv - n_vars:]
    s_vals = [F.mle(inv_s, sp), F.mle(s_field, sp)]
    t_vals = [F.mle(m_field, tp), F.mle(inv_t, tp), F.mle(t_field, tp)]
    _open(s_vals, sp, tr)
    _open(t_vals, tp, tr)
    return {"beta": beta, "beta_retries": retries, "alpha": alpha, "u": u,
            "rounds": [tuple(r) for r in rounds], "final_values": tuple(finals),
            "point": point, "secret_values": tuple(s_vals), "table_values": tuple(t_vals)}
