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
