"""Host-side lookup-table generation (restates zklora.tables, tables.py:40-117).

Entries are tuples, computed once per process (lru_cache): the scalar
float64 loop is kept exactly as the reference's (a vectorised np.exp may
round differently in the last bit), so it is not cheap.

Table values come from float64 host code in the reference (np.exp, math.exp,
math.sqrt with round-half-away, quantize.py:81-85).  They are generated here
with the same scalar operations in the same order (SURVEY.md sec. 7 hard
part 8: never recompute them on the device), then uploaded as int32 device
columns.  tests/test_host.py pins every table against the reference's own
output (tests/golden/tables_g4096.json).
"""

import functools
import math

import numpy as np


def round_half_away(x):
    """quantize.py:81-85."""
    if x >= 0:
        return int(np.floor(x + 0.5))
    return -int(np.floor(-x + 0.5))


def _silu_real(x):  # tables.py:40-42 (0-d float64 array, as the reference calls it)
    x = np.asarray(x, dtype=np.float64)
    return x / (1.0 + np.exp(-x))


def _silu_deriv_real(x):  # tables.py:45-48
    x = np.asarray(x, dtype=np.float64)
    s = 1.0 / (1.0 + np.exp(-x))
    return s * (1.0 + x * (1.0 - s))


@functools.lru_cache(maxsize=None)
def silu_entries(gamma, act_bound):
    """tables.py:65-69, 92-95: x in [-act*gamma, act*gamma)."""
    half = act_bound * gamma
    xs = range(-half, half)
    return tuple(xs), tuple(round_half_away(gamma * float(_silu_real(x / gamma))) for x in xs)


@functools.lru_cache(maxsize=None)
def silu_deriv_entries(gamma, act_bound):
    """tables.py:72-76, 98-101."""
    half = act_bound * gamma
    xs = range(-half, half)
    return tuple(xs), tuple(round_half_away(gamma * float(_silu_deriv_real(x / gamma)))
                            for x in xs)


@functools.lru_cache(maxsize=None)
def exp_segment_entries(gamma, radices, k):
    """tables.py:56-62, 86-89: digit -> round(gamma * exp(-digit * base_k / gamma))."""
    base = 1
    for r in radices[:k]:
        base *= r
    xs = range(radices[k])
    return tuple(xs), tuple(round_half_away(gamma * math.exp(-d * (base / gamma))) for d in xs)


@functools.lru_cache(maxsize=None)
def rsqrt_entries(gamma, act_bound, eps):
    """tables.py:79-83, 104-106: x in [0, act*gamma)."""
    xs = range(act_bound * gamma)
    return tuple(xs), tuple(round_half_away(gamma / math.sqrt(x / gamma + eps)) for x in xs)


def quant_range(gamma, act_bound):
    """tables.py:109-111: (first value, size)."""
    return -act_bound * gamma, 2 * act_bound * gamma


def residue_range(zeta):
    """tables.py:114-117."""
    return -(zeta // 2), zeta


def radix_bases(radices):
    """quantize.py:111-118: base_k = product of the radices before position k."""
    bases, acc = [], 1
    for b in radices:
        bases.append(acc)
        acc *= b
    return bases


def exp_segment_value(gamma, radices, k, digit):
    """tables.py:56-62 for one digit."""
    if not 0 <= digit < radices[k]:
        raise KeyError("digit %d outside segment %d" % (digit, k))
    base = radix_bases(radices)[k]
    return round_half_away(gamma * math.exp(-digit * (base / gamma)))
