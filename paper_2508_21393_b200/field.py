"""Prime fields of the prover and the GPU batch inversion.

Mirrors pkg/src/zklora/field.py (MODULUS, TEST_MODULUS, InversionOfZero,
inverse, batch_inverse).  batch_inverse runs on the GPU (zkl_batch_inverse,
hierarchical Montgomery trick) and keeps the reference's error behaviour
exactly (field.py:34-46): a literal 0 entry raises "cannot invert 0 at index
i" for the first such i; an entry that is a non-zero multiple of p makes the
reference fail later, on the final inversion, with "cannot invert 0".
"""

import ctypes

from . import _native as N
from . import device as D

MODULUS = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
TEST_MODULUS = (1 << 61) - 1


class InversionOfZero(ZeroDivisionError):
    """Raised when a multiplicative inverse of zero is requested."""


def element_size(modulus):
    return 8 if modulus.bit_length() <= 64 else 32


def inverse(value, modulus):
    """Scalar inverse (host; one exponentiation)."""
    value %= modulus
    if value == 0:
        raise InversionOfZero("cannot invert 0")
    return pow(value, modulus - 2, modulus)


_INV_POW2 = {}


def inverse_pow2(k, modulus):
    """2^-k mod p = ((p + 1) / 2)^k (p odd): a k-step power instead of a
    full-length exponentiation (~0.1 ms in Python), cached -- it sits on the
    per-claim host path of every zkMat (gadgets.py:246) and lookup ratio."""
    key = (k, modulus)
    v = _INV_POW2.get(key)
    if v is None:
        v = pow((modulus + 1) // 2, k, modulus)
        _INV_POW2[key] = v
    return v


def to_signed(value, modulus):
    return value if value <= modulus // 2 else value - modulus


def from_signed(value, modulus):
    return value % modulus


def batch_inverse_device(buf, n, spec, add=None, out=None):
    """In-device batch inversion: out[i] = 1 / (buf[i] + add).

    Returns (out, first_zero) where first_zero is None or the first index
    whose input is zero (then `out` is undefined).
    """
    lib = N.lib()
    if out is None:
        out = D.empty(spec, n)
    fz = ctypes.c_int64(-1)
    rc = lib.zkl_batch_inverse(spec.fid, D.ptr(out), D.ptr(buf), n,
                               D.scalar_bytes(add, spec) if add is not None else None,
                               ctypes.byref(fz), D.stream())
    if rc == N.ZKL_ERR_ZERO:
        return out, fz.value
    N.check(rc)
    return out, None


def batch_inverse(values, modulus):
    """Drop-in for zklora.field.batch_inverse (field.py:34-46), on the GPU."""
    values = list(values)
    if not values:
        return []
    spec = D.spec_for(modulus)
    buf = D.upload(values, spec)
    out, fz = batch_inverse_device(buf, len(values), spec)
    if fz is not None:
        try:
            first_raw = values.index(0)
        except ValueError:
            first_raw = None
        if first_raw is not None:
            raise InversionOfZero("cannot invert 0 at index %d" % first_raw)
        raise InversionOfZero("cannot invert 0")
    return D.download(out, spec, len(values))
