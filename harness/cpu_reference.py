"""The reference's CPU prover, timed (bench.py's reference arm and its
cpu_baseline leg).  MEASUREMENT HARNESS ONLY: nothing in the package imports
it, and nothing here is on the measured GPU path.

* `ref_zkmat_sample`: the REAL reference (baseline/_ref, the unmodified
  zklora package) proving a corner of the cfg2 X.W claim exactly as
  prove_matmul does (gadgets.py:241-251: r_u / r_v, the four replicated
  tables, prove_sumcheck sumcheck.py:98-130), single-threaded pure Python.
* `ref_lookup_ladder`: the real reference prove_lookup (lookup.py:143-251,
  commitments replaced by the deterministic stub on its side, as in
  tests/golden/make_golden.py) on a doubling ladder of Eq.-7 claim sizes; the
  per-table-entry cost is fitted and extrapolated to cfg3's 7 x 2^25 claim
  (labelled as extrapolated).
* `factored_cpu_cfg2`: the oracle's factored zkMat restatement (numpy
  matvecs, oracle/zkmat.py) over the full cfg2 step, so the algorithmic
  factor (factored vs replicated claim) and the hardware factor (B200 vs
  host cores) can be read apart.
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
P_BIG = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


def reference_available():
    return os.path.isdir(os.path.join(REF, "zklora"))


def _zklora():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import zklora.gadgets as G
    import zklora.lookup as L
    import zklora.mle as M
    import zklora.sumcheck as S
    import zklora.transcript as T

    return G, L, M, S, T


def corner(X, W, dims):
    """The (d0, d1, d2) corner of X.W: X[:2^d0, :2^d1], W[:2^d1, :2^d2], C."""
    d0, d1, d2 = dims
    a = X[: 1 << d0, : 1 << d1].astype(np.int64)
    b = W[: 1 << d1, : 1 << d2].astype(np.int64)
    return a, b, a @ b


def ref_zkmat_sample(a, b, c, dims, seed=b"sample"):
    """(field elements of the claim, seconds): the reference's own zkMat
    sumcheck on the given integer matrices."""
    G, _, M, S, T = _zklora()
    p = P_BIG
    d0, d1, d2 = dims
    A = [int(v) % p for v in a.reshape(-1)]
    B = [int(v) % p for v in b.reshape(-1)]
    C = [int(v) % p for v in c.reshape(-1)]
    t0 = time.perf_counter()
    tr = T.Transcript(b"zklora-b200/cpu", p, seed)
    r_u = tr.challenge_vector(b"matmul/r_u", d0)
    r_v = tr.challenge_vector(b"matmul/r_v", d2)
    tables = G._replicated_tables(A, B, C, M.eq_table(r_u, p), M.eq_table(r_v, p), d0, d1, d2, p)
    terms = [S.Term(1, (0, 1, 2)), S.Term((-G.inverse(1 << d1, p)) % p, (0, 3))]
    S.prove_sumcheck(S.SumcheckClaim(0, list(tables), terms, 3, p), tr)
    return 4 * (1 << sum(dims)), time.perf_counter() - t0


class _StubCom:
    def __init__(self, num_vars):
        self.num_vars = num_vars

    def serialize(self, group):
        return b"zkl-stub/v1" + bytes([self.num_vars])


def _install_stub(G, L, M):
    def commit(key, table, blinding=None):
        return _StubCom((len(table) - 1).bit_length())

    def open_batch(key, tables, blindings, point, tr, rng):
        vals = [M.mle_evaluate(list(t), list(point), tr.modulus) for t in tables]
        for r in point:
            tr.append(b"open/point", r)
        for y in vals:
            tr.append(b"open/value", y)
        return vals, None

    L.commit, L.open_batch = commit, open_batch


def ref_lookup_sample(d_log, n_log, seed=0):
    """(claim elements 7 * max(d, n), seconds) of one reference prove_lookup
    with stub commitments (commitment time excluded)."""
    G, L, M, S, T = _zklora()
    _install_stub(G, L, M)
    from types import SimpleNamespace

    p = P_BIG
    rng = np.random.default_rng(seed)
    n = 1 << n_log
    table = tuple(int(v) for v in rng.integers(0, 1 << 40, size=n))
    secret = tuple(table[int(i)] for i in rng.integers(0, n, size=1 << d_log))
    tab = L.LookupTable(table, _StubCom(n_log))
    sec = L.SecretVector(secret, _StubCom(d_log), ())
    key = SimpleNamespace(group=None)
    rngv = SimpleNamespace(vector=lambda k: [0] * k)
    t0 = time.perf_counter()
    mult = L.compute_multiplicities(secret, tab)
    L.prove_lookup(sec, mult, tab, key, T.Transcript(b"zklora-b200/cpu", p, b"lk"), rngv)
    return 7 * max(1 << d_log, n), time.perf_counter() - t0


def ref_lookup_ladder(n_log=10, d_logs=(12, 13, 14)):
    """Fit seconds = a + b * elements over a doubling ladder of reference
    prove_lookup runs; returns the points and the per-element cost."""
    pts = [ref_lookup_sample(d, n_log, seed=d) for d in d_logs]
    x = np.array([e for e, _ in pts], dtype=np.float64)
    y = np.array([s for _, s in pts], dtype=np.float64)
    b, a = np.polyfit(x, y, 1)
    return {"points": [{"field_elems": int(e), "seconds": s} for e, s in pts],
            "fit_s_per_elem": float(b), "fit_intercept_s": float(a)}


def factored_cpu_cfg2(claims_host):
    """Seconds for the oracle's factored zkMat restatement (numpy, exact
    integer matvecs) over every claim of one cfg2 step; the same transcript
    traffic and outputs as the GPU prover."""
    from oracle import fs, zkmat

    t0 = time.perf_counter()
    for name, a, b, c, dims in claims_host:
        zkmat.prove_factored(a.astype(np.int64).reshape(-1), b.astype(np.int64).reshape(-1),
                             c.reshape(-1), dims, fs.FS(b"zklora-b200/cpu", P_BIG, name.encode()))
    return time.perf_counter() - t0


def ref_commit_sample(n_log=12, seed=0):
    """Seconds per committed entry of the reference's Hyrax row-Pedersen
    commitment (commit.py:97-115: one multi-exponentiation per row in the
    ~262-bit Schnorr group of group.py:69-76), with a real CommitmentKey.
    Commitments are outside the optimisation target (BASELINE north star:
    "timed separately"); this is that timing, on the host."""
    _zklora()
    import zklora.commit as C
    import zklora.group as GR

    group = GR.group_for_modulus(P_BIG)
    key = C.keygen(n_log, b"zklora-b200/commit-timing", group)
    rng = np.random.default_rng(seed)
    table = [int(v) % P_BIG for v in rng.integers(-2 ** 15, 2 ** 15, size=1 << n_log)]
    t0 = time.perf_counter()
    C.commit(key, table)
    sec = time.perf_counter() - t0
    return {"entries": 1 << n_log, "seconds": sec, "s_per_entry": sec / (1 << n_log)}
