"""Prime-field constants and inversion (oracle restatement).

Follows /root/reference/pkg/src/zklora/field.py:9-46.
"""

# BLS12-381 scalar field order (field.py:9)
P_BIG = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
# Mersenne test field (field.py:12)
P_TEST = (1 << 61) - 1


class ZeroInverse(ZeroDivisionError):
    """Oracle analogue of zklora.field.InversionOfZero (field.py:15)."""


def width(p):
    """Serialized element width, field.py:18-20: 8 bytes if p < 2^64 else 32."""
    return 8 if p.bit_length() <= 64 else 32


def inv(x, p):
    """Fermat inverse; field.py:24-31 (gmpy2 absent -> pow fallback)."""
    x %= p
    if not x:
        raise ZeroInverse("cannot invert 0")
    return pow(x, p - 2, p)


def batch_inv(xs, p):
    """Montgomery trick, field.py:34-46.

    The zero check runs in the forward prefix pass, so the reported index is
    the first zero in input order.
    """
    n = len(xs)
    run = [1] * (n + 1)
    for k in range(n):
        if xs[k] == 0:
            raise ZeroInverse("cannot invert 0 at index %d" % k)
        run[k + 1] = run[k] * xs[k] % p
    acc = inv(run[n], p)
    res = [0] * n
    for k in reversed(range(n)):
        res[k] = run[k] * acc % p
        acc = acc * xs[k] % p
    return res
