"""Non-linear gadget provers (oracle restatement, test infrastructure only).

Follows /root/reference/pkg/src/zklora/gadgets.py:
  _absorb_operands   gadgets.py:183-186
  _prove_pair_lookup gadgets.py:679-688 (x + alpha*y compression, tables.py:131-140)
  prove_rescale      gadgets.py:600-622
  prove_swiglu       gadgets.py:761-782
  prove_rsqrt        gadgets.py:842-847
Operands are committed tensors with the deterministic stub commitment
(stubcommit.py); values are canonical residues.  Nothing in the product
imports this module.
"""

from . import logup
from .stubcommit import stub_bytes


def digest(rv, cv):
    """TensorRef.digest for a committed operand (gadgets.py:89-97)."""
    return b"com:" + bytes([rv, cv]) + stub_bytes(rv + cv)


def absorb_operands(tr, tag, shapes):
    tr.append(b"gadget/tag", tag)
    for rv, cv in shapes:
        tr.append(b"gadget/operand", digest(rv, cv))


def _log2(n):
    return (n - 1).bit_length()


def lookup(secret, shape, table, tr, be):
    """prove_lookup(secret_vector, compute_multiplicities(...), table) for a
    committed tensor of `shape` against a committed single-column table."""
    mult = logup.multiplicities(secret, table)
    return logup.prove(secret, mult, table, stub_bytes(_log2(len(table))),
                       stub_bytes(sum(shape)), tr, be)


def pair_lookup(label, x, y, shape, tx, ty, tr, be):
    p = tr.modulus
    tr.append(label + b"/x", digest(*shape))
    tr.append(label + b"/y", digest(*shape))
    alpha = tr.challenge(label + b"/alpha")
    secret = [(a + alpha * b) % p for a, b in zip(x, y)]
    table = [(a + alpha * b) % p for a, b in zip(tx, ty)]
    return lookup(secret, shape, table, tr, be)


def rescale(wide, narrow, resid, shape, divisor, zeta, quant_range, residue_range, tr, be):
    if divisor <= 0 or zeta % divisor:
        raise ValueError("divisor must divide zeta")
    absorb_operands(tr, b"rescale", [shape] * 3)
    tr.append(b"rescale/divisor", divisor)
    point = tr.challenge_vector(b"rescale/point", sum(shape))
    identity = be.open([wide, narrow, resid], point, tr)
    q = lookup(narrow, shape, quant_range, tr, be)
    r = lookup(resid, shape, residue_range, tr, be)
    return {"identity": identity, "lookups": [q, r]}


def swiglu(wide, out, narrow, resid, shape, mode, pair, residue_range, tr, be):
    if mode not in ("phi", "phi_prime"):
        raise ValueError("mode must be phi or phi_prime")
    absorb_operands(tr, b"swiglu", [shape] * 2)
    tr.append(b"swiglu/mode", mode.encode())
    absorb_operands(tr, b"swiglu/wit", [shape] * 2)
    point = tr.challenge_vector(b"swiglu/point", sum(shape))
    identity = be.open([wide, narrow, resid], point, tr)
    act = pair_lookup(b"swiglu/act", narrow, out, shape, pair[0], pair[1], tr, be)
    r = lookup(resid, shape, residue_range, tr, be)
    return {"identity": identity, "lookups": [act, r]}


def rsqrt(v, u, shape, pair, tr, be):
    absorb_operands(tr, b"rsqrt", [shape] * 2)
    return {"lookups": [pair_lookup(b"rsqrt/pair", v, u, shape, pair[0], pair[1], tr, be)]}
