"""logUp lookup argument core (oracle restatement).

Follows /root/reference/pkg/src/zklora/lookup.py:91-318.  Commitments are
out of scope for this repo; they are injected through ``backend`` (see
``stubcommit``) exactly where the reference calls commit / open_batch /
verify_batch, so the transcript sees the same byte stream on both sides.
"""

from .multilinear import eq_at, eq_vec, evaluate, zero_prefix
from .prime import batch_inv, inv
from .sc import combine, prove as sc_prove, verify as sc_verify

MAX_RETRIES = 3  # lookup.py:44


class NotInTable(ValueError):
    def __init__(self, index, value):
        super().__init__("secret entry %d (value %d) not in table" % (index, value))
        self.index = index
        self.value = value


class Pole(RuntimeError):
    pass


def multiplicities(secret, table):
    """lookup.py:91-99; duplicate table values resolve to their LAST index."""
    where = {}
    for j, v in enumerate(table):
        where[v] = j
    counts = [0] * len(table)
    for i, s in enumerate(secret):
        j = where.get(s)
        if j is None:
            raise NotInTable(i, s)
        counts[j] += 1
    return counts


def logup_terms(alpha, ratio, p):
    """lookup.py:116-126; factor order eq, A, S+b, ind, B, T+b, m."""
    a2 = alpha * alpha % p
    a3 = a2 * alpha % p
    return [
        (alpha, (0, 1, 2)),
        ((-alpha) % p, (0, 3)),
        (a2, (0, 4, 5)),
        (a3, (1,)),
        ((-a3 * ratio) % p, (6, 4)),
    ]


def lifted_tables(secret, inv_s, table, inv_t, mult, u, beta, p):
    """lookup.py:188-202: pad (d <= n) or replicate (d > n)."""
    d, n = len(secret), len(table)
    if d <= n:
        pad = n - d
        a_full = list(inv_s) + [0] * pad
        s_full = list(secret) + [0] * pad
        ind = [1] * d + [0] * pad
        b_full, t_full, m_full = list(inv_t), list(table), list(mult)
    else:
        c = d // n
        a_full, s_full, ind = list(inv_s), list(secret), [1] * d
        b_full, t_full, m_full = list(inv_t) * c, list(table) * c, list(mult) * c
    return [
        eq_vec(u, p),
        a_full,
        [(s + beta) % p for s in s_full],
        ind,
        b_full,
        [(t + beta) % p for t in t_full],
        m_full,
    ]


def prove(secret, mult, table, table_com, secret_com, tr, backend):
    """lookup.py:143-251 with commitments delegated to ``backend``.

    Returns a dict whose keys mirror LookupProof (lookup.py:102-113) plus the
    challenges for debugging.
    """
    p = tr.modulus
    d, n = len(secret), len(table)
    if d == 0 or d & (d - 1):
        raise ValueError("secret length must be a power of two")
    if len(mult) != n:
        raise ValueError("multiplicity vector must match the table size")
    m_com = backend.commit(list(mult))
    tr.append(b"lookup/table", table_com)
    tr.append(b"lookup/secret", secret_com)
    tr.append(b"lookup/mult", m_com)

    poles = {(-s) % p for s in secret} | {(-t) % p for t in table}
    retries = 0
    beta = tr.challenge(b"lookup/beta")
    while beta in poles:
        retries += 1
        if retries > MAX_RETRIES:
            raise Pole("challenge hit a pole %d times" % retries)
        tr.append(b"lookup/beta-retry", retries)
        beta = tr.challenge(b"lookup/beta")

    inv_s = batch_inv([(beta + s) % p for s in secret], p)
    inv_t = batch_inv([(beta + t) % p for t in table], p)
    a_com = backend.commit(inv_s)
    b_com = backend.commit(inv_t)
    tr.append(b"lookup/inv-secret", a_com)
    tr.append(b"lookup/inv-table", b_com)

    alpha = tr.challenge(b"lookup/alpha")
    big = max(d, n)
    nv = (big - 1).bit_length()
    u = tr.challenge_vector(b"lookup/u", nv)
    ratio = inv(big // n, p)
    tabs = lifted_tables(secret, inv_s, table, inv_t, mult, u, beta, p)
    rounds, finals, point = sc_prove(alpha * alpha % p, tabs, logup_terms(alpha, ratio, p), 3, tr)

    d_vars = (d - 1).bit_length()
    n_vars = (n - 1).bit_length()
    s_pt = point[nv - d_vars :]
    t_pt = point[nv - n_vars :]
    s_vals = backend.open([inv_s, list(secret)], s_pt, tr)
    t_vals = backend.open([list(mult), inv_t, list(table)], t_pt, tr)
    return {
        "secret_vars": d_vars,
        "beta_retries": retries,
        "multiplicity_commitment": m_com,
        "inverse_secret_commitment": a_com,
        "inverse_table_commitment": b_com,
        "rounds": rounds,
        "final_values": finals,
        "secret_values": tuple(s_vals),
        "table_values": tuple(t_vals),
        "point": point,
        "beta": beta,
        "alpha": alpha,
        "u": u,
    }


def verify(secret_com, table, table_com, proof, tr, backend):
    """lookup.py:254-318 (opening checks delegated to ``backend``)."""
    p = tr.modulus
    n = len(table)
    d_vars = proof["secret_vars"]
    n_vars = (n - 1).bit_length()
    nv = max(d_vars, n_vars)
    if proof["beta_retries"] > MAX_RETRIES:
        return False
    tr.append(b"lookup/table", table_com)
    tr.append(b"lookup/secret", secret_com)
    tr.append(b"lookup/mult", proof["multiplicity_commitment"])
    beta = tr.challenge(b"lookup/beta")
    for k in range(proof["beta_retries"]):
        tr.append(b"lookup/beta-retry", k + 1)
        beta = tr.challenge(b"lookup/beta")
    tr.append(b"lookup/inv-secret", proof["inverse_secret_commitment"])
    tr.append(b"lookup/inv-table", proof["inverse_table_commitment"])
    alpha = tr.challenge(b"lookup/alpha")
    u = tr.challenge_vector(b"lookup/u", nv)
    ratio = inv((1 << nv) // n, p)
    terms = logup_terms(alpha, ratio, p)
    ok, point, expected = sc_verify(alpha * alpha % p, terms, 3, nv, proof["rounds"], tr)
    if not ok:
        return False
    s_pt = point[nv - d_vars :]
    t_pt = point[nv - n_vars :]
    if not backend.check(list(proof["secret_values"]), s_pt, tr):
        return False
    if not backend.check(list(proof["table_values"]), t_pt, tr):
        return False
    a_o, s_o = proof["secret_values"]
    m_o, b_o, t_o = proof["table_values"]
    gap = nv - d_vars
    pre = zero_prefix(point, gap, p) if gap else 1
    vals = [
        eq_at(u, point, p),
        pre * a_o % p,
        (pre * s_o + beta) % p,
        pre,
        b_o,
        (t_o + beta) % p,
        m_o,
    ]
    return combine(terms, vals, p) == expected


def mle(t, pt, p):
    return evaluate(t, pt, p)
