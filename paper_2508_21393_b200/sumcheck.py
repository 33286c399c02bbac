"""Sumcheck prover on the GPU, drop-in for zklora.sumcheck.prove_sumcheck.

Mirrors pkg/src/zklora/sumcheck.py: the claim / proof types (Term,
SumcheckClaim with the same validation, RoundPolynomial, SumcheckProof),
``prove_sumcheck(claim, tr) -> (SumcheckProof, point)`` with the same
transcript traffic, and a host verifier with the reference's semantics.

The round loop runs on the device: one fused kernel per round folds every
table by the previous challenge and evaluates the round polynomial at
x = 0..degree (zkl_sumcheck_round); only the (degree+1) evaluations cross to
the host, where the Fiat-Shamir transcript draws the next challenge.
"""

import ctypes
from dataclasses import dataclass

from . import _native as N
from . import device as D
from .field import inverse


class DegreeOverflow(ValueError):
    pass


class SumcheckError(ValueError):
    pass


@dataclass(frozen=True)
class Term:
    coefficient: int
    factors: tuple


@dataclass
class SumcheckClaim:
    """Same fields and validation as sumcheck.py:32-56."""

    claimed_sum: int
    tables: list
    terms: list
    degree: int
    modulus: int

    def __post_init__(self):
        if self.degree > 3:
            raise DegreeOverflow("per-variable degree above 3 unsupported")
        for t in self.terms:
            if len(t.factors) > self.degree:
                raise DegreeOverflow(
                    "term with %d factors exceeds degree %d" % (len(t.factors), self.degree))
        sizes = {len(t) for t in self.tables}
        if len(sizes) != 1:
            raise SumcheckError("factor tables must share one variable count")
        size = sizes.pop()
        if size & (size - 1):
            raise SumcheckError("table length must be a power of two")

    @property
    def num_vars(self):
        return (len(self.tables[0]) - 1).bit_length()


@dataclass(frozen=True)
class RoundPolynomial:
    evaluations: tuple


@dataclass
class SumcheckProof:
    rounds: list
    final_values: tuple


# Result classes; install() points these at the reference's classes so proofs
# serialize with the reference's wire format (serialize.py:52-74).
TYPES = {"RoundPolynomial": RoundPolynomial, "SumcheckProof": SumcheckProof}


def combine(terms, values, modulus):
    """sumcheck.py:70-78 (host, scalar)."""
    total = 0
    for t in terms:
        prod = t.coefficient
        for idx in t.factors:
            prod = prod * values[idx] % modulus
        total = (total + prod) % modulus
    return total


def absorb_claim(tr, claimed_sum, terms, degree, num_vars):
    """sumcheck.py:90-95."""
    tr.append(b"sumcheck/sum", claimed_sum)
    tr.append(b"sumcheck/shape", bytes([degree, num_vars, len(terms)]))
    for t in terms:
        tr.append(b"sumcheck/coeff", t.coefficient)
        tr.append(b"sumcheck/factors", bytes(t.factors))


class _TermArgs:
    """ctypes views of a term list for zkl_sumcheck_round."""

    def __init__(self, terms, spec):
        nt = len(terms)
        if nt > 8:
            raise NotImplementedError("GPU sumcheck supports at most 8 terms (got %d)" % nt)
        self.nt = nt
        self.nf = (ctypes.c_int32 * max(nt, 1))(*[len(f) for _, f in terms])
        flat = []
        for _, f in terms:
            flat.extend(list(f) + [0] * (3 - len(f)))
        self.fi = (ctypes.c_int32 * max(3 * nt, 3))(*flat)
        self.coeffs = D.scalars_bytes([c for c, _ in terms], spec) or b"\0" * spec.nbytes


def native_transcript(tr, spec):
    """True when `tr` is a reference-semantics Transcript whose state the
    native driver can advance (this package's or zklora's own class)."""
    st = getattr(tr, "state", None)
    if not isinstance(st, (bytes, bytearray)) or len(st) != 64:
        return False
    if getattr(tr, "modulus", None) != spec.modulus or NATIVE_TRANSCRIPT is False:
        return False
    app = getattr(type(tr), "append", None)
    from .transcript import Transcript

    if app is Transcript.append:
        return True
    return (getattr(app, "__qualname__", "") == "Transcript.append"
            and type(tr).__module__.endswith("transcript"))


NATIVE_TRANSCRIPT = True  # tests flip this to exercise the per-round host path


def _decode(raw, nb, count, _fb=int.from_bytes):
    raw = bytes(raw)
    return [_fb(raw[i:i + nb], "little") for i in range(0, nb * count, nb)]


def run_rounds(spec, tables, num_vars, terms, degree, tr, post_add=None, post_mul=None):
    """Run every round of a device-resident claim.

    tables: list of device field vectors (each 2^num_vars entries, consumed).
    terms: list of (coefficient int, factor tuple).
    post_add: per-round ints or None; post_mul: int or None (1):
    evals[x] = post_mul * (post_add[j] + sum_x).
    Returns (rounds as tuples, point, finals) with finals canonical ints.
    """
    lib = N.lib()
    k = len(tables)
    if k > 8:
        raise NotImplementedError("GPU sumcheck supports at most 8 tables (got %d)" % k)
    ta = _TermArgs(terms, spec)
    ptrs = (ctypes.c_void_p * k)(*[t.data_ptr() for t in tables])
    nb = spec.nbytes
    strm = D.stream()
    if num_vars == 0:
        return [], [], [D.read_scalar(t, spec) for t in tables]
    addb = D.scalars_bytes(post_add, spec) if post_add is not None else None
    mulb = D.scalar_bytes(post_mul, spec) if post_mul is not None else None
    if native_transcript(tr, spec):
        state = ctypes.create_string_buffer(bytes(tr.state), 64)
        rbuf = (ctypes.c_uint8 * (num_vars * (degree + 1) * nb))()
        pbuf = (ctypes.c_uint8 * (num_vars * nb))()
        fbuf = (ctypes.c_uint8 * (k * nb))()
        N.check(lib.zkl_sumcheck_prove(spec.fid, ptrs, k, num_vars, degree, ta.nt, ta.nf, ta.fi,
                                       ta.coeffs, addb, mulb, state, rbuf, pbuf, fbuf, strm))
        flat = _decode(bytes(rbuf), nb, num_vars * (degree + 1))
        rounds = [tuple(flat[j * (degree + 1):(j + 1) * (degree + 1)]) for j in range(num_vars)]
        tr.state = state.raw[:64]
        log = getattr(tr, "log", None)
        if log is not None:
            log.extend((b"sumcheck/eval", (e.bit_length() + 7) // 8 or 1) for e in flat)
        return rounds, _decode(bytes(pbuf), nb, num_vars), _decode(bytes(fbuf), nb, k)
    # generic transcript object: per-round host loop
    evbuf = (ctypes.c_uint8 * (4 * nb))()
    rounds, point = [], []
    size = 1 << num_vars
    r_prev = None
    for j in range(num_vars):
        ab = addb[j * nb:(j + 1) * nb] if addb is not None else None
        rb = D.scalar_bytes(r_prev, spec) if r_prev is not None else None
        N.check(lib.zkl_sumcheck_round(spec.fid, ptrs, k, size, 1 if rb else 0, rb, degree,
                                       ta.nt, ta.nf, ta.fi, ta.coeffs, ab, mulb, evbuf, strm))
        if rb:
            size >>= 1
        evals = tuple(_decode(bytes(evbuf), nb, degree + 1))
        rounds.append(evals)
        for e in evals:
            tr.append(b"sumcheck/eval", e)
        r_prev = tr.challenge(b"sumcheck/round")
        point.append(r_prev)
    fin = (ctypes.c_uint8 * (k * nb))()
    N.check(lib.zkl_sumcheck_finish(spec.fid, ptrs, k, D.scalar_bytes(r_prev, spec), fin, strm))
    return rounds, point, _decode(bytes(fin), nb, k)


def prove_sumcheck(claim, tr):
    """Drop-in for zklora.sumcheck.prove_sumcheck (sumcheck.py:98-130)."""
    p = claim.modulus
    degree = claim.degree
    n = claim.num_vars
    spec = D.spec_for(p)
    for t in claim.terms:
        for idx in t.factors:
            if n and not 0 <= idx < len(claim.tables):
                raise IndexError("list index out of range")
    absorb_claim(tr, claim.claimed_sum, claim.terms, degree, n)
    if n == 0:
        # no rounds: the reference returns the raw single entries
        return TYPES["SumcheckProof"]([], tuple(t[0] for t in claim.tables)), []
    dev = [D.upload(list(t), spec) for t in claim.tables]
    terms = [(t.coefficient, tuple(t.factors)) for t in claim.terms]
    rounds, point, finals = run_rounds(spec, dev, n, terms, degree, tr)
    RP = TYPES["RoundPolynomial"]
    return TYPES["SumcheckProof"]([RP(e) for e in rounds], tuple(finals)), point
