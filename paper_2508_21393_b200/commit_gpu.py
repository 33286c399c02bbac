"""Hyrax row commitments on the GPU.

`commit(key, table, blinding=None)` is zklora.commit.commit (commit.py:98-115):
the 2^n table laid out as split_shape(n) rows x cols, row i committed as the
Pedersen product h^{b_i} prod_j g_j^{t[i cols + j]} in the key's Schnorr
group (group.py:64-70), the same group elements bit for bit.  The
multi-exponentiation runs in libzkl_b200.so (csrc/commit.cu): fixed-base byte
windows per generator, built once per key and cached on the device, then one
table product per nonzero exponent byte.

    from paper_2508_21393_b200 import commit_gpu
    com = commit_gpu.commit(key, table)          # a zklora Commitment
"""

import ctypes

import numpy as np
import torch

from . import _native as N
from . import device as D
from .device import MODULUS, TEST_MODULUS

# group id, element bytes, exponent words per scalar field
_GROUPS = {MODULUS: (0, 33, 8), TEST_MODULUS: (1, 9, 2)}


def supports(key):
    """True for the Schnorr groups the GPU implements (group.py:64-67)."""
    g = key.group
    o = _GROUPS.get(g.order)
    return o is not None and g.q == {MODULUS: 96 * MODULUS + 1,
                                     TEST_MODULUS: 52 * TEST_MODULUS + 1}[g.order]


def _split_shape(num_vars):
    row_vars = (num_vars + 1) // 2
    return 1 << row_vars, 1 << (num_vars - row_vars)


class _KeyTables:
    __slots__ = ("key_id", "width", "buf", "group", "qbytes", "ewords")

    def __init__(self, key):
        group = key.group
        gid, qbytes, ewords = _GROUPS[group.order]
        gens = list(key.generators) + [key.blinding_generator]
        raw = b"".join(int(g).to_bytes(qbytes, "little") for g in gens)
        nbytes = N.lib().zkl_commit_table_bytes(gid, len(gens))
        self.buf = torch.empty(int(nbytes), dtype=torch.uint8, device="cuda")
        N.check(N.lib().zkl_commit_tables(gid, raw, len(gens), D.ptr(self.buf), D.stream()))
        self.key_id = id(key)
        self.width = len(key.generators)
        self.group, self.qbytes, self.ewords = gid, qbytes, ewords


_TABLES = {}


def key_tables(key):
    """The device window tables of a key (built on first use, then cached;
    the cache key names the key's generators)."""
    gens = key.generators
    ident = (id(key), key.seed, len(gens), key.group.q, gens[0], gens[-1],
             key.blinding_generator)
    t = _TABLES.get(ident)
    if t is None:
        if len(_TABLES) >= 8:
            _TABLES.clear()
        t = _TABLES[ident] = _KeyTables(key)
    return t


def _exponents(values, count, modulus, ewords):
    """Canonical exponents as device words: a list of residues, or a
    DeviceVector (storage form, converted on the device)."""
    if isinstance(values, D.DeviceVector):
        spec = values.spec
        out = D.empty(spec, count)
        N.check(N.lib().zkl_from_mont(spec.fid, D.ptr(out), D.ptr(values.buf), count, D.stream()))
        return out
    vals = list(values)
    if len(vals) != count:
        raise ValueError("table length does not match the layout")
    raw = np.frombuffer(D.encode(vals, D.spec_for(modulus)), dtype=np.uint8)
    return torch.from_numpy(raw.copy()).to("cuda")


def commit_rows(key, table, num_vars, blinding=None):
    """Row elements (ints) of the commitment to a 2^num_vars table."""
    kt = key_tables(key)
    rows, cols = _split_shape(num_vars)
    if cols > kt.width:
        raise _ref("commit").KeyTooSmall("key supports %d columns, need %d" % (kt.width, cols))
    modulus = key.group.order
    vals = _exponents(table, rows * cols, modulus, kt.ewords)
    blind = None
    if blinding is not None:
        blinding = list(blinding)
        if len(blinding) != rows:
            raise _ref("commit").DimensionMismatch("need %d blinding scalars" % rows)
        blind = _exponents(blinding, rows, modulus, kt.ewords)
    out = (ctypes.c_uint8 * (rows * kt.qbytes))()
    N.check(N.lib().zkl_commit_rows(kt.group, D.ptr(kt.buf), cols, D.ptr(vals),
                                    D.ptr(blind) if blind is not None else None, kt.width,
                                    rows, out, D.stream()))
    raw = bytes(out)
    q = kt.qbytes
    return tuple(int.from_bytes(raw[i * q:(i + 1) * q], "little") for i in range(rows))


def commit_row(key, values, blinding):
    """One Pedersen row h^blinding prod_j g_j^values[j] (commit.py:87-95
    `_row_commit`) as a group element."""
    kt = key_tables(key)
    cols = len(values)
    if cols > kt.width:
        raise _ref("commit").KeyTooSmall("key supports %d columns, need %d" % (kt.width, cols))
    modulus = key.group.order
    vals = _exponents(values, cols, modulus, kt.ewords)
    blind = _exponents([blinding], 1, modulus, kt.ewords) if blinding else None
    out = (ctypes.c_uint8 * kt.qbytes)()
    N.check(N.lib().zkl_commit_rows(kt.group, D.ptr(kt.buf), cols, D.ptr(vals),
                                    D.ptr(blind) if blind is not None else None, kt.width,
                                    1, out, D.stream()))
    return int.from_bytes(bytes(out), "little")


def open_batch(key, tables, blindings, point, tr, rng):
    """Drop-in for zklora.commit.open_batch (commit.py:150-215): the same
    values, transcript records and OpeningProof, with the table-sized work on
    the GPU -- each table's row-combined vector left^T T is a field matvec,
    the batch combination is linear in those vectors, and the sigma proof's
    row commitment is one GPU multi-exponentiation.  `tables` may be lists of
    residues or DeviceVectors."""
    from .gadgets import DeviceMatrix, _axpy, _matvec

    cm = _ref("commit")
    modulus = tr.modulus
    spec = D.spec_for(modulus)
    group = key.group
    num_vars = len(point)
    rows, cols = _split_shape(num_vars)
    for t in tables:
        if len(t) != rows * cols:
            raise cm.DimensionMismatch("table does not match point arity")
    half = (num_vars + 1) // 2
    left = D.eq_table(list(point[:half]), spec)
    right = D.eq_table(list(point[half:]), spec)
    # y_k = left^T T_k (cols), value_k = <y_k, right>
    ys, values = [], []
    for t in tables:
        buf = D.field_buffer(t, spec)
        M = DeviceMatrix(buf.view(-1)[: rows * cols * spec.words].view(rows * cols, spec.words),
                         rows, cols, N.MT_FIELD, spec)
        y = _matvec(M, left, True, spec)
        ys.append(y)
        values.append(D.dot(y, right, spec, cols))
    for r in point:
        tr.append(b"open/point", r)
    for v in values:
        tr.append(b"open/value", v)
    batch = tr.challenge(b"open/batch") if len(tables) > 1 else 1
    # t_vec = left^T (sum_k batch^k T_k) = sum_k batch^k y_k; the blinding alike
    t_vec = ys[0]
    coeff = batch
    for y in ys[1:]:
        t_vec = _axpy(t_vec, coeff, y, cols, spec)
        coeff = coeff * batch % modulus
    blind = [0] * rows
    coeff = 1
    for b in blindings:
        if b is not None:
            for i, x in enumerate(b):
                blind[i] = (blind[i] + coeff * x) % modulus
        coeff = coeff * batch % modulus
    b_comb = D.dot(left, D.upload(blind, spec), spec, rows)
    y_comb = D.dot(t_vec, right, spec, cols)
    nonce = rng.vector(cols)
    nonce_blind = rng.next()
    blinded_row = commit_row(key, nonce, nonce_blind)
    nonce_dev = D.upload(nonce, spec)
    blinded_value = D.dot(nonce_dev, right, spec, cols)
    tr.append(b"open/sigma", group.encode(blinded_row))
    tr.append(b"open/sigma-value", blinded_value)
    c = tr.challenge(b"open/challenge")
    responses = tuple(D.download(_axpy(nonce_dev, c, t_vec, cols, spec), spec, cols))
    blinding_response = (nonce_blind + c * b_comb) % modulus
    return values, cm.OpeningProof(y_comb, blinded_row, blinded_value, responses,
                                   blinding_response)


def _ref(name):
    """The reference package's module (its Commitment and error types)."""
    import importlib

    return importlib.import_module("zklora.%s" % name)


def commit(key, table, blinding=None):
    """Drop-in for zklora.commit.commit (commit.py:98-115) on the GPU."""
    cm = _ref("commit")
    n = len(table)
    num_vars = (n - 1).bit_length()
    if n != 1 << num_vars:
        raise ValueError("table length must be a power of two")
    return cm.Commitment(num_vars, commit_rows(key, table, num_vars, blinding))
