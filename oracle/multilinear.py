"""Multilinear-extension helpers (oracle restatement).

Follows /root/reference/pkg/src/zklora/mle.py:50-100.  The first variable
is the most significant index bit everywhere.
"""


def fold_msb(t, r, p):
    """mle.py:50-56: bind the MSB variable: t'[i] = (1-r) t[i] + r t[i+h]."""
    h = len(t) >> 1
    s = (1 - r) % p
    return [(s * t[i] + r * t[h + i]) % p for i in range(h)]


def evaluate(t, pt, p):
    """mle.py:59-64: evaluation by successive folds."""
    cur = list(t)
    for r in pt:
        cur = fold_msb(cur, r, p)
    return cur[0]


def eq_vec(pt, p):
    """mle.py:67-82: eq(pt, x) over the cube; pt[0] pairs with the MSB."""
    cur = [1]
    for r in pt:
        r %= p
        s = (1 - r) % p
        nxt = []
        for v in cur:
            nxt.append(v * s % p)
            nxt.append(v * r % p)
        cur = nxt
    return cur


def eq_at(a, b, p):
    """mle.py:85-92."""
    assert len(a) == len(b)
    out = 1
    for x, y in zip(a, b):
        out = out * ((x * y + (1 - x) * (1 - y)) % p) % p
    return out


def zero_prefix(pt, count, p):
    """mle.py:95-100."""
    out = 1
    for r in pt[:count]:
        out = out * ((1 - r) % p) % p
    return out
