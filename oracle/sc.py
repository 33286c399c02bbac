"""Generic product sumcheck (oracle restatement).

Follows /root/reference/pkg/src/zklora/sumcheck.py:25-172.  Claims are
plain tuples here: ``terms`` is a list of (coefficient, factor-index tuple).
The prover returns (rounds, final_values, point) with rounds a list of
evaluation tuples at x = 0..degree.
"""

from .multilinear import fold_msb
from .prime import inv


def combine(terms, vals, p):
    """sumcheck.py:70-78."""
    acc = 0
    for coef, factors in terms:
        v = coef
        for f in factors:
            v = v * vals[f] % p
        acc = (acc + v) % p
    return acc


def absorb_claim(tr, claimed_sum, terms, degree, n):
    """sumcheck.py:90-95: the claim is bound before the first round."""
    tr.append(b"sumcheck/sum", claimed_sum)
    tr.append(b"sumcheck/shape", bytes([degree, n, len(terms)]))
    for coef, factors in terms:
        tr.append(b"sumcheck/coeff", coef)
        tr.append(b"sumcheck/factors", bytes(factors))


def num_vars_of(tables):
    return (len(tables[0]) - 1).bit_length()


def round_evals(tables, terms, degree, p):
    """One round's evaluations, sumcheck.py:110-123 (g(1) computed directly)."""
    h = len(tables[0]) >> 1
    out = [0] * (degree + 1)
    for i in range(h):
        lo = [t[i] for t in tables]
        hi = [t[i + h] for t in tables]
        step = [(b - a) % p for a, b in zip(lo, hi)]
        cur = lo
        for x in range(degree + 1):
            if x == 1:
                cur = hi
            elif x >= 2:
                cur = [(c + s) % p for c, s in zip(cur, step)]
            out[x] = (out[x] + combine(terms, cur, p)) % p
    return out


def prove(claimed_sum, tables, terms, degree, tr):
    """sumcheck.py:98-130."""
    p = tr.modulus
    cur = [list(t) for t in tables]
    n = num_vars_of(cur)
    absorb_claim(tr, claimed_sum, terms, degree, n)
    rounds, point = [], []
    for _ in range(n):
        ev = round_evals(cur, terms, degree, p)
        rounds.append(tuple(ev))
        for e in ev:
            tr.append(b"sumcheck/eval", e)
        r = tr.challenge(b"sumcheck/round")
        point.append(r)
        cur = [fold_msb(t, r, p) for t in cur]
    return rounds, tuple(t[0] for t in cur), point


def lagrange(ev, x, p):
    """sumcheck.py:133-145."""
    d = len(ev) - 1
    acc = 0
    for j, y in enumerate(ev):
        num = den = 1
        for k in range(d + 1):
            if k != j:
                num = num * ((x - k) % p) % p
                den *= j - k
        acc = (acc + y * num % p * inv(den % p, p)) % p
    return acc


def verify(claimed_sum, terms, degree, n, rounds, tr):
    """sumcheck.py:148-172 -> (ok, point, expected_final)."""
    p = tr.modulus
    if len(rounds) != n:
        return False, [], 0
    absorb_claim(tr, claimed_sum, terms, degree, n)
    running = claimed_sum % p
    point = []
    for ev in rounds:
        if len(ev) != degree + 1 or (ev[0] + ev[1]) % p != running:
            return False, [], 0
        for e in ev:
            tr.append(b"sumcheck/eval", e)
        r = tr.challenge(b"sumcheck/round")
        point.append(r)
        running = lagrange(ev, r, p)
    return True, point, running
