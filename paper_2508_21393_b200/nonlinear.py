"""Device-resident non-linear gadget provers: rescale, SwiGLU, rsqrt.

Mirrors of zklora.gadgets (reference gadgets.py):
  prove_rescale  gadgets.py:600-622  (quotient + residue range lookups)
  prove_swiglu   gadgets.py:761-782  (activation pair lookup + residue lookup)
  prove_rsqrt    gadgets.py:842-847  (pair lookup)
with the same transcript traffic, argument meaning and exceptions.  They
exist so that tensors that live on the GPU as int16/int32/int64 matrices
(DeviceMatrix) are proven without ever building Python lists: range-table
lookups bin their integer secrets by offset (the secret is lifted to field
elements only if a path needs it), pair lookups compress on the device, and
the logUp sumchecks run on the round engine (lookup.py).  With host
ProverTensors they behave like the reference functions (which, once
install() has run, already reach this backend through prove_lookup).

Tables: `TableSet` holds the same fields as tables.py:156-168; its single
column tables may carry DeviceVector entries and its pair tables int32
device columns (`device_range_table`, `device_pair_table`).
"""

from dataclasses import dataclass

import torch

from . import _native as N
from . import device as D
from .commit_stub import attach
from .gadgets import ShapeMismatch, _absorb_operands, _open_tables, prove_pair_lookup
from .lookup import (LookupTable, SecretVector, compute_multiplicities, multiplicities_indexed,
                     multiplicities_range, prove_lookup)


class RangeViolation(ValueError):
    """gadgets.py RangeViolation (witness outside a table domain)."""


class DigitOutOfRange(ValueError):
    """quantize.py DigitOutOfRange (shifted exponent outside [0, xi))."""


class NormalizationBudgetExceeded(ValueError):
    """gadgets.py NormalizationBudgetExceeded (softmax row sum drift)."""


@dataclass(frozen=True)
class PairTable:
    """tables.py:120-153: aligned (input, output) columns."""

    x: LookupTable
    y: LookupTable
    name: str

    @property
    def size(self):
        return self.x.size


@dataclass(frozen=True)
class TableSet:
    """tables.py:156-168 (the fields the gadgets read)."""

    params: object
    eps: float
    modulus: int
    digest: bytes
    exp_segments: tuple
    silu: PairTable
    silu_deriv: PairTable
    rsqrt: PairTable
    quant_range: LookupTable
    residue_range: LookupTable


@dataclass
class RescaleProof:
    tag = "rescale"
    divisor: int
    shape: tuple
    identity_opening: object
    quant_lookup: object
    resid_lookup: object


@dataclass
class SwigluProof:
    tag = "swiglu"
    mode: str
    shape: tuple
    narrow_ref: object
    resid_ref: object
    identity_opening: object
    activation_lookup: object
    resid_lookup: object


@dataclass
class RsqrtProof:
    tag = "rsqrt"
    shape: tuple
    lookup: object


@dataclass
class SoftmaxRowProof:
    tag = "softmax_row"
    num_vars: int
    xi_prime: int
    digit_refs: tuple
    partial_refs: tuple
    chain_wide_refs: tuple
    chain_narrow_refs: tuple
    chain_resid_refs: tuple
    decomposition_opening: object
    digit_lookups: tuple
    chain_prod_proofs: tuple
    chain_rescale_proofs: tuple
    normalization_opening: object


TYPES = {"RescaleProof": RescaleProof, "SwigluProof": SwigluProof, "RsqrtProof": RsqrtProof,
         "SoftmaxRowProof": SoftmaxRowProof,
         "NormalizationBudgetExceeded": NormalizationBudgetExceeded}


# ---------------------------------------------------------------------------
def device_range_table(lo, n, spec, commitment, name):
    """A consecutive-integer single-column table [lo, lo+n) lifted on the GPU
    (quant_range_entries / residue_range_entries, tables.py:109-117)."""
    col = torch.arange(lo, lo + n, dtype=torch.int32, device="cuda")
    t = LookupTable(D.DeviceVector(D.lift(col, spec), n, spec), attach(commitment, col), name)
    object.__setattr__(t, "int_column", col)  # lets multiplicities bin by offset
    return t


def device_pair_table(xs, ys, commitment_x, commitment_y, name):
    """A pair table with int32 device columns (tables.py:208-214)."""
    tx = torch.as_tensor(xs, dtype=torch.int32).cuda()
    ty = torch.as_tensor(ys, dtype=torch.int32).cuda()
    return PairTable(LookupTable(tx, attach(commitment_x, tx), name + ".x"),
                     LookupTable(ty, attach(commitment_y, ty), name + ".y"), name)


def rescale_witness_device(wide, divisor, params):
    """rescale_witness (gadgets.py:563-580) for a signed int device tensor:
    (narrow int16, resid int16 = r * zeta/divisor), one kernel pass
    (zkl_rescale_witness).  A quotient outside the quant_range domain raises
    RangeViolation like the reference (gadgets.py:575); nothing is clamped."""
    import ctypes

    zeta = params.zeta
    if divisor <= 0 or zeta % divisor:
        raise ValueError("divisor must divide zeta")
    half = params.act_bound * params.gamma_fp
    w = wide.contiguous()
    q = torch.empty(w.shape, dtype=torch.int16, device=w.device)
    r = torch.empty(w.shape, dtype=torch.int16, device=w.device)
    fb, nb = ctypes.c_int64(-1), ctypes.c_uint64(0)
    rc = N.lib().zkl_rescale_witness(D.ptr(w), D._INT_TYPES[w.dtype], w.numel(), divisor,
                                     zeta // divisor, -half, half - 1, D.ptr(q), D.ptr(r),
                                     ctypes.byref(fb), ctypes.byref(nb), D.stream())
    if rc == N.ZKL_ERR_MISSING:
        bad = int(w.reshape(-1)[fb.value])
        q0 = (bad + divisor // 2) // divisor
        raise RangeViolation("rescale quotient %d outside table domain (%d entries)"
                             % (q0, nb.value))
    N.check(rc)
    return q, r


def _int_matrix(pt):
    dev = getattr(pt, "device", None)
    if dev is not None and dev.mtype != N.MT_FIELD:
        return dev.t
    return None


def _range_lookup(pt, table, key, tr, rng):
    """prove_lookup(pt.as_secret_vector(), compute_multiplicities(...), table)
    (gadgets.py:606-613) for a committed operand."""
    if pt.ref.kind != "committed":
        raise ValueError("public operands have no secret vector")
    col = _int_matrix(pt)
    if col is not None and isinstance(table.entries, D.DeviceVector):
        spec = table.entries.spec
        flat = col.reshape(-1)
        secret = SecretVector(D.LiftedColumn(flat, spec), pt.ref.commitment,
                              tuple(pt.blinding))
        got = None
        tcol = getattr(table, "int_column", None)
        if tcol is not None:  # the table is exactly the range tcol[0] .. tcol[0]+n-1
            got = multiplicities_range(secret.entries, table, flat, tcol)
        counts, index = got if got is not None else multiplicities_indexed(secret.entries, table)
        return prove_lookup(secret, counts, table, key, tr, rng, secret_index=index)
    secret = SecretVector(tuple(pt.flat()), pt.ref.commitment, tuple(pt.blinding))
    return prove_lookup(secret, compute_multiplicities(secret.entries, table), table, key, tr,
                        rng)


def _shape(pt):
    return (pt.ref.row_vars, pt.ref.col_vars)


def prove_rescale(wide, narrow, resid, divisor, tables, key, tr, rng):
    """Drop-in for zklora.gadgets.prove_rescale (gadgets.py:600-622): proves
    (zeta/div)*wide = zeta*narrow + resid with narrow in quant_range and
    resid in residue_range."""
    zeta = tables.params.zeta
    if divisor <= 0 or zeta % divisor:
        raise ValueError("divisor must divide zeta")
    shape = _shape(wide)
    for t in (narrow, resid):
        if _shape(t) != shape:
            raise ShapeMismatch("rescale operands must share a shape")
    _absorb_operands(tr, b"rescale", [wide.ref, narrow.ref, resid.ref], key.group)
    tr.append(b"rescale/divisor", divisor)
    point = tr.challenge_vector(b"rescale/point", wide.ref.num_vars)
    identity_opening = _open_tables(key, [wide, narrow, resid], point, tr, rng)
    quant_lookup = _range_lookup(narrow, tables.quant_range, key, tr, rng)
    resid_lookup = _range_lookup(resid, tables.residue_range, key, tr, rng)
    return TYPES["RescaleProof"](divisor=divisor, shape=shape, identity_opening=identity_opening,
                                 quant_lookup=quant_lookup, resid_lookup=resid_lookup)


def prove_swiglu(wide, out, narrow, resid, mode, tables, key, tr, rng):
    """Drop-in for zklora.gadgets.prove_swiglu (gadgets.py:761-782): proves
    out = activation(round(wide / zeta)) with a ranged residue."""
    if mode not in ("phi", "phi_prime"):
        raise ValueError("mode must be phi or phi_prime")
    shape = _shape(wide)
    for t in (out, narrow, resid):
        if _shape(t) != shape:
            raise ShapeMismatch("swiglu operands must share a shape")
    pair = tables.silu if mode == "phi" else tables.silu_deriv
    _absorb_operands(tr, b"swiglu", [wide.ref, out.ref], key.group)
    tr.append(b"swiglu/mode", mode.encode())
    _absorb_operands(tr, b"swiglu/wit", [narrow.ref, resid.ref], key.group)
    point = tr.challenge_vector(b"swiglu/point", wide.ref.num_vars)
    identity_opening = _open_tables(key, [wide, narrow, resid], point, tr, rng)
    activation_lookup = prove_pair_lookup(b"swiglu/act", narrow, out, pair, key, tr, rng)
    resid_lookup = _range_lookup(resid, tables.residue_range, key, tr, rng)
    return TYPES["SwigluProof"](mode=mode, shape=shape, narrow_ref=narrow.ref,
                                resid_ref=resid.ref, identity_opening=identity_opening,
                                activation_lookup=activation_lookup, resid_lookup=resid_lookup)


def prove_rsqrt(v, u, tables, key, tr, rng):
    """Drop-in for zklora.gadgets.prove_rsqrt (gadgets.py:842-847)."""
    if _shape(u) != _shape(v):
        raise ShapeMismatch("rsqrt operands must share a shape")
    _absorb_operands(tr, b"rsqrt", [v.ref, u.ref], key.group)
    lookup = prove_pair_lookup(b"rsqrt/pair", v, u, tables.rsqrt, key, tr, rng)
    return TYPES["RsqrtProof"](shape=_shape(v), lookup=lookup)


# ---------------------------------------------------------------------------
# softmax (one row): gadgets.py:878-1036
def softmax_row_witness(z_row, params, modulus):
    """Host restatement of gadgets.py:878-922 (float64 host code, like the
    reference: SURVEY.md sec. 7 hard part 8).  Returns (xi_prime, digits[k][i],
    partials[k][i], chain [(wide, narrow, resid)], p_row) as signed ints."""
    import math

    from .tables import exp_segment_value, radix_bases, round_half_away

    radices = tuple(params.radices)
    if len(radices) < 2:
        raise ValueError("softmax needs at least two radix positions")
    if len(z_row) & (len(z_row) - 1):
        raise ShapeMismatch("softmax rows must have power-of-two length")
    g, zeta = params.gamma_fp, params.zeta
    m = max(z_row)
    total = sum(math.exp((z - m) / g) for z in z_row)
    xi_prime = m + round_half_away(g * math.log(total))
    bases = radix_bases(radices)
    digits, partials = [], []
    for z in z_row:
        v = xi_prime - z
        if v < 0 or v >= params.xi:
            raise DigitOutOfRange("shifted exponent %d outside [0, xi)" % v)
        ds, rest = [], v
        for b in radices:  # quantize.py:121-135, least significant first
            ds.append(rest % b)
            rest //= b
        if rest:
            raise DigitOutOfRange("value %d exceeds the radix capacity" % v)
        digits.append(ds)
        partials.append([exp_segment_value(g, radices, k, d) for k, d in enumerate(ds)])
    kc = len(radices)
    digit_cols = [[digits[i][k] for i in range(len(z_row))] for k in range(kc)]
    partial_cols = [[partials[i][k] for i in range(len(z_row))] for k in range(kc)]
    chain, current = [], list(partial_cols[0])
    for k in range(1, kc):
        wide = [c * y for c, y in zip(current, partial_cols[k])]
        narrow = [(w + zeta // 2) // zeta for w in wide]
        resid = [w - zeta * q for w, q in zip(wide, narrow)]
        chain.append((wide, narrow, resid))
        current = narrow
    return xi_prime, digit_cols, partial_cols, chain, current


def normalization_budget(row_len, params):
    """gadgets.py:925-927."""
    return row_len * (len(params.radices) + 1)


def _committed_vector(values, key, rng, dtype=torch.int32):
    """commit_tensor (gadgets.py:120-128) of a 1 x len(values) signed vector
    as a device operand under the stub key."""
    from .gadgets import DeviceMatrix, ProverTensor, TensorRef, commit_backend

    n = (len(values) - 1).bit_length()
    be = commit_backend(key)
    rows, _ = be.split_shape(n)
    blinding = tuple(rng.vector(rows))
    t = torch.tensor(values, dtype=dtype, device="cuda").view(1, -1)
    return ProverTensor(None, TensorRef("committed", 0, n, commitment=be.commit_size(n)), blinding,
                        device=DeviceMatrix.from_int_tensor(t))


def prove_softmax_row(z_row, p_row, witness, tables, key, tr, rng):
    """Drop-in for zklora.gadgets.prove_softmax_row (gadgets.py:930-1036):
    digit decomposition opening, one exp pair lookup per radix position, the
    product chain (elementprod + rescale per step), the half-point
    normalisation opening with its drift budget.  Witness columns become
    device operands (stub commitments) when z_row lives on the GPU."""
    from types import SimpleNamespace

    from .gadgets import ProverTensor, TensorRef, commit_backend, prove_elementprod
    from .field import inverse

    p = tr.modulus
    params = tables.params
    xi_prime, digit_cols, partial_cols, chain, final = witness
    n = z_row.ref.num_vars
    row_len = 1 << n
    if p_row.ref.num_vars != n:
        raise ShapeMismatch("probability row shape differs from score row")
    kc = len(params.radices)
    be = commit_backend(key)
    device = getattr(z_row, "device", None) is not None and be.__name__.endswith("commit_stub")
    if device:
        got = p_row.device.t.reshape(-1).tolist() if getattr(p_row, "device", None) is not None \
            else None
    else:
        from .field import to_signed

        got = [to_signed(v, p) for v in p_row.flat()]
    if got is not None and [int(v) for v in got] != [int(v) for v in final]:
        raise ValueError("p_row does not match the witness chain output")

    def vec(values):
        if device:
            dtype = torch.int64 if max(abs(int(v)) for v in values) >= (1 << 31) else torch.int32
            return _committed_vector(values, key, rng, dtype)
        rows, _ = be.split_shape(n)
        blinding = tuple(rng.vector(rows))
        entries = [int(v) % p for v in values]
        com = be.commit(key, entries, list(blinding) if blinding else None)
        return ProverTensor(SimpleNamespace(data=entries), TensorRef("committed", 0, n,
                                                                     commitment=com), blinding)

    digit_ts = [vec(digit_cols[k]) for k in range(kc)]
    partial_ts = [vec(partial_cols[k]) for k in range(kc)]
    wide_ts, narrow_ts, resid_ts = [], [], []
    for idx, (wide, narrow, resid) in enumerate(chain):
        wide_ts.append(vec(wide))
        narrow_ts.append(p_row if idx == len(chain) - 1 else vec(narrow))
        resid_ts.append(vec(resid))

    _absorb_operands(tr, b"softmax", [z_row.ref, p_row.ref], key.group)
    tr.append(b"softmax/xi", xi_prime % p)
    for t in digit_ts + partial_ts + wide_ts + narrow_ts[:-1] + resid_ts:
        tr.append(b"softmax/witness", t.ref.digest(key.group))
    rho = tr.challenge_vector(b"softmax/decomp", n)
    decomposition_opening = _open_tables(key, digit_ts + [z_row], rho, tr, rng)
    digit_lookups = tuple(
        prove_pair_lookup(b"softmax/exp%d" % k, digit_ts[k], partial_ts[k],
                          tables.exp_segments[k], key, tr, rng)
        for k in range(kc))
    chain_prod_proofs, chain_rescale_proofs = [], []
    current = partial_ts[0]
    for idx in range(len(chain)):
        chain_prod_proofs.append(
            prove_elementprod(current, partial_ts[idx + 1], wide_ts[idx], key, tr, rng))
        chain_rescale_proofs.append(
            prove_rescale(wide_ts[idx], narrow_ts[idx], resid_ts[idx], params.zeta, tables, key,
                          tr, rng))
        current = narrow_ts[idx]
    half = inverse(2, p)
    normalization_opening = _open_tables(key, [p_row], [half] * n, tr, rng)
    total = (1 << n) * normalization_opening.values[0] % p
    drift = total - params.gamma_fp
    drift = (drift + p // 2) % p - p // 2  # to_signed
    if abs(drift) > normalization_budget(row_len, params):
        raise TYPES["NormalizationBudgetExceeded"](
            "row sum off by %d units (budget %d)" % (drift, normalization_budget(row_len, params)))
    return TYPES["SoftmaxRowProof"](
        num_vars=n, xi_prime=xi_prime, digit_refs=tuple(t.ref for t in digit_ts),
        partial_refs=tuple(t.ref for t in partial_ts),
        chain_wide_refs=tuple(t.ref for t in wide_ts),
        chain_narrow_refs=tuple(t.ref for t in narrow_ts[:-1]),
        chain_resid_refs=tuple(t.ref for t in resid_ts),
        decomposition_opening=decomposition_opening, digit_lookups=digit_lookups,
        chain_prod_proofs=tuple(chain_prod_proofs),
        chain_rescale_proofs=tuple(chain_rescale_proofs),
        normalization_opening=normalization_opening)
