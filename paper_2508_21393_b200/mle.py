"""MLE helpers on the GPU: drop-ins for zklora.mle (mle.py:50-100).

Variable order as in the reference: the first coordinate is the most
significant index bit; matrices are row bits || column bits.
"""

import ctypes

from . import _native as N
from . import device as D


class DimensionMismatch(ValueError):
    pass


def fold_table(table, r, modulus):
    """mle.py:50-56 on the device."""
    spec = D.spec_for(modulus)
    half = len(table) // 2
    if half == 0:
        return []
    src = D.upload(list(table), spec)
    dst = D.empty(spec, half)
    N.check(N.lib().zkl_fold(spec.fid, D.ptr(dst), D.ptr(src), half, D.scalar_bytes(r, spec),
                             D.stream()))
    return D.download(dst, spec, half)


def eq_table(point, modulus):
    """mle.py:67-82 on the device."""
    spec = D.spec_for(modulus)
    return D.download(D.eq_table(list(point), spec), spec, 1 << len(point))


def mle_evaluate_device(buf, n_vars, point, spec):
    """MLE of a device field vector (2^n_vars entries) at `point` by folds."""
    if len(point) != n_vars:
        raise DimensionMismatch("point has %d coordinates, polynomial has %d variables"
                                % (len(point), n_vars))
    lib = N.lib()
    if n_vars == 0:
        return D.read_scalar(buf, spec)
    size = 1 << n_vars
    tmp = D.empty(spec, size // 2)
    src = buf
    for r in point:  # first fold out of place (keeps buf), then in place
        half = size // 2
        N.check(lib.zkl_fold(spec.fid, D.ptr(tmp), D.ptr(src), half, D.scalar_bytes(r, spec),
                             D.stream()))
        src = tmp
        size = half
    return D.read_scalar(tmp, spec)


def mle_evaluate(table, point, modulus):
    """mle.py:59-64 on the device."""
    spec = D.spec_for(modulus)
    n = (len(table) - 1).bit_length()
    return mle_evaluate_device(D.upload(list(table), spec), n, list(point), spec)


def mle_evaluate_matrix(M, point, spec):
    """MLE of an integer DeviceMatrix (row bits || column bits) at `point`:
    eq(point_rows)^T (M eq(point_cols)), one matrix-vector pass over the
    integers (zkl_matvec) instead of lifting 2^n entries to field elements."""
    from .gadgets import _matvec

    rv, cv = (M.rows - 1).bit_length(), (M.cols - 1).bit_length()
    if rv + cv != len(point):
        raise DimensionMismatch("point has %d coordinates, polynomial has %d variables"
                                % (len(point), rv + cv))
    y = _matvec(M, D.eq_table(point[rv:], spec), False, spec)
    return D.dot(D.eq_table(point[:rv], spec), y, spec, M.rows)


def mle_evaluate_many(tables, point, modulus):
    """mle_evaluate_any for several tables at one point (an opening batch,
    commit.py:192-195): integer matrices of one shape share the two eq
    tables."""
    spec = D.spec_for(modulus)
    point = list(point)
    out, shared = [], {}
    for t in tables:
        if getattr(t, "mtype", N.MT_FIELD) != N.MT_FIELD:
            rv = (t.rows - 1).bit_length()
            if rv + (t.cols - 1).bit_length() != len(point):
                raise DimensionMismatch("point has %d coordinates, matrix has %d variables"
                                        % (len(point), rv + (t.cols - 1).bit_length()))
            if rv not in shared:
                shared[rv] = (D.eq_table(point[rv:], spec), D.eq_table(point[:rv], spec))
            ec, er = shared[rv]
            from .gadgets import _matvec

            out.append(D.dot(er, _matvec(t, ec, False, spec), spec, t.rows))
        else:
            out.append(mle_evaluate_any(t, point, modulus))
    return out


def mle_evaluate_any(table, point, modulus):
    """Python list or DeviceMatrix / device vector."""
    spec = D.spec_for(modulus)
    if getattr(table, "mtype", N.MT_FIELD) != N.MT_FIELD:
        return mle_evaluate_matrix(table, list(point), spec)
    lifted = getattr(table, "as_field_vector", None)
    if lifted is not None:
        return mle_evaluate_device(lifted(spec), len(point), list(point), spec)
    return mle_evaluate(table, point, modulus)


def eq_eval(u, x, modulus):
    """mle.py:85-92 (scalar, host)."""
    if len(u) != len(x):
        raise DimensionMismatch("eq kernel arity mismatch")
    acc = 1
    for a, b in zip(u, x):
        acc = acc * ((a * b + (1 - a) * (1 - b)) % modulus) % modulus
    return acc


def zero_prefix_eval(point, count, modulus):
    """mle.py:95-100 (scalar, host)."""
    acc = 1
    for r in point[:count]:
        acc = acc * ((1 - r) % modulus) % modulus
    return acc
