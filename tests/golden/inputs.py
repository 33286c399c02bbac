"""Deterministic input generators shared by make_golden.py and the tests.

No dependency on the reference or on the product: plain numpy PCG64 streams,
so the GPU box regenerates exactly the inputs the goldens were made from.
"""

import numpy as np

P_BIG = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
P_TEST = (1 << 61) - 1


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def uniform_int(seed, shape, lo, hi):
    """Uniform signed ints in [lo, hi] as an int64 numpy array."""
    return rng(seed).integers(lo, hi + 1, size=shape, dtype=np.int64)


def next_pow2(x):
    return 1 if x <= 1 else 1 << (x - 1).bit_length()


def padded(mat):
    """Zero-pad a 2-D int array to power-of-two shape (quantize.py:176-183)."""
    r, c = mat.shape
    out = np.zeros((next_pow2(r), next_pow2(c)), dtype=np.int64)
    out[:r, :c] = mat
    return out


def matmul_case(seed, rows, inner, cols, lo=-32768, hi=32767, tamper=None):
    """A (rows x inner), B (inner x cols), C = A B exact; padded, int64.

    tamper = (i, j, delta) perturbs C[i, j] after the product.
    """
    a = uniform_int(seed, (rows, inner), lo, hi)
    b = uniform_int(seed + 1, (inner, cols), lo, hi)
    c = (a.astype(object) @ b.astype(object)).astype(np.int64)
    if tamper is not None:
        i, j, delta = tamper
        c[i, j] += delta
    return padded(a), padded(b), padded(c)


def to_field(arr, p):
    """Signed ints -> canonical residues (negatives as p - |x|, field.py:54-55)."""
    return [int(v) % p for v in np.asarray(arr).reshape(-1).tolist()]


def field_vec(seed, n, p):
    g = rng(seed)
    # 4 x 64-bit words per element, reduced mod p
    words = g.integers(0, 2**63, size=(n, 4), dtype=np.int64).tolist()
    out = []
    for w in words:
        v = 0
        for k, x in enumerate(w):
            v |= int(x) << (64 * k)
        out.append(v % p)
    return out
