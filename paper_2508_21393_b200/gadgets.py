"""zkMat and elementprod provers on the GPU (drop-ins for zklora.gadgets).

prove_matmul (gadgets.py:230-265) emits the reference's (d0+d1+d2)-round
replicated-table sumcheck (gadgets.py:210-251) bit for bit, but never builds
its four 2^(d0+d1+d2) tables.  The claim
    sum_{u,w,v} eq(r_u,u) eq(r_v,v) [A(u,w) B(w,v) - 2^-d1 C(u,v)] = 0
is proven phase by phase over MLE partial evaluations (DESIGN.md,
"Factored zkMat"):
  U (d0 rounds): two-factor sumcheck of (E_u, h), h = A (B E_v) - (C E_v)
  W (d1 rounds): E_hat [ sum a(w) bv(w) - 2^-d1 2^rem kappa ],
                 a = E(rho_u)^T A, bv = B E_v, kappa = <E(rho_u)^T C, E_v>
  V (d2 rounds): E_hat sum E_v(v) [alpha_s bw(v) - 2^-d1 cu(v)],
                 bw = E(rho_w)^T B, cu = E(rho_u)^T C
Every matrix is read twice (one row product, one column product) by the
wide-accumulator matvec kernels; every phase runs on the dense round engine.
Operands may be the reference's ProverTensor (field residues on the host)
or DeviceMatrix (int16 / int32 / int64 / field matrices already on the GPU).
"""

import ctypes
from dataclasses import dataclass

import torch

from . import _native as N
from . import device as D
from . import shard
from .field import inverse_pow2
from .sumcheck import TYPES as SC_TYPES
from .sumcheck import Term, absorb_claim, native_transcript, run_rounds


class ShapeMismatch(ValueError):
    pass


@dataclass(frozen=True)
class TensorRef:
    """Mirror of gadgets.py:56-97 (verifier-side operand handle)."""

    kind: str
    row_vars: int
    col_vars: int
    commitment: object = None
    value: int = 0

    @property
    def num_vars(self):
        return self.row_vars + self.col_vars

    def digest(self, group):
        head = bytes([self.row_vars, self.col_vars])
        if self.kind == "committed":
            return b"com:" + head + self.commitment.serialize(group)
        return self.kind.encode() + b":" + head + self.value.to_bytes(32, "little", signed=False)


class DeviceMatrix:
    """A padded row-major matrix resident on the GPU.

    mtype: N.MT_I16 / MT_I32 / MT_I64 (signed integers, value = x mod p) or
    N.MT_FIELD (storage-form field elements, W int64 words per entry).
    """

    def __init__(self, tensor, rows, cols, mtype, spec=None):
        self.t = tensor
        self.rows, self.cols, self.mtype, self.spec = rows, cols, mtype, spec
        self._field = None

    @classmethod
    def from_int_tensor(cls, t):
        t = t.contiguous()
        mt = {torch.int16: N.MT_I16, torch.int32: N.MT_I32, torch.int64: N.MT_I64}[t.dtype]
        r, c = t.shape
        return cls(t, r, c, mt)

    @classmethod
    def from_field_list(cls, values, rows, cols, spec):
        return cls(D.upload(list(values), spec), rows, cols, N.MT_FIELD, spec)

    def as_field_vector(self, spec):
        if self.mtype == N.MT_FIELD:
            return self.t
        if self._field is None:
            self._field = D.lift(self.t.view(-1), spec)
        return self._field


@dataclass(frozen=True)
class ProverTensor:
    """Mirror of gadgets.py:100-113 with an optional device-resident copy."""

    tensor: object
    ref: TensorRef
    blinding: tuple = ()
    device: object = None  # DeviceMatrix

    def flat(self):
        return list(self.tensor.data)


@dataclass
class Opening:
    values: tuple
    proof: object


@dataclass
class MatmulProof:
    tag = "matmul"
    dims: tuple
    sumcheck: object
    a_opening: object
    b_opening: object
    c_opening: object


@dataclass
class ElementprodProof:
    tag = "elementprod"
    shape: tuple
    c_opening: object
    sumcheck: object
    ab_opening: object


@dataclass
class MataddProof:
    tag = "matadd"
    sign: int
    shape: tuple
    opening: object


TYPES = {"Opening": Opening, "MatmulProof": MatmulProof, "ElementprodProof": ElementprodProof,
         "MataddProof": MataddProof}


# ---------------------------------------------------------------------------
def commit_backend(key):
    """zklora.commit for real keys, the stub for StubKey (commit_stub.py)."""
    if getattr(key, "is_stub", False):
        from . import commit_stub

        return commit_stub
    import zklora.commit as zc  # the reference's own commitment path

    return zc


def _absorb_operands(tr, tag, refs, group):
    """gadgets.py:183-186."""
    tr.append(b"gadget/tag", tag)
    for ref in refs:
        tr.append(b"gadget/operand", ref.digest(group))


def _open_tables(key, prover_tensors, point, tr, rng, values=None):
    """gadgets.py:160-167 through the commitment backend."""
    be = commit_backend(key)
    tables, blindings = [], []
    for pt in prover_tensors:
        dev = getattr(pt, "device", None)
        tables.append(dev if (dev is not None and be.__name__.endswith("commit_stub"))
                      else pt.flat())
        rows, _ = be.split_shape(pt.ref.num_vars)
        blindings.append(list(pt.blinding) if pt.blinding else [0] * rows)
    if values is not None and be.__name__.endswith("commit_stub"):
        vals, proof = be.open_batch(key, tables, blindings, point, tr, rng, values=values)
    else:
        vals, proof = be.open_batch(key, tables, blindings, point, tr, rng)
    return TYPES["Opening"](tuple(vals), proof)


def _device_matrix(pt, rows, cols, spec):
    dev = getattr(pt, "device", None)
    if dev is not None:
        return dev
    return DeviceMatrix.from_field_list(pt.flat(), rows, cols, spec)


# ---------------------------------------------------------------------------
_MT_BYTES = {N.MT_I16: 2, N.MT_I32: 4, N.MT_I64: 8}


def _matvec(M, x, transpose, spec):
    out = D.empty(spec, M.cols if transpose else M.rows)
    N.check(N.lib().zkl_matvec(spec.fid, M.mtype, D.ptr(M.t), M.rows, M.cols,
                               1 if transpose else 0, D.ptr(x), D.ptr(out), D.stream()))
    return out


def _axpy(a, k, b, n, spec):
    out = D.empty(spec, n)
    N.check(N.lib().zkl_axpy(spec.fid, D.ptr(out), D.ptr(a), D.scalar_bytes(k, spec),
                             D.ptr(b), n, D.stream()))
    return out


NATIVE_DRIVER = True  # tests flip this to exercise the Python phase driver


def _matmul_native(A, B, C, dims, tr, spec):
    """zkl_matmul_prove: the whole claim in one C call (csrc/zkmat.cu)."""
    d0, d1, d2 = dims
    n = d0 + d1 + d2
    nb = spec.nbytes
    state = ctypes.create_string_buffer(bytes(tr.state), 64)
    rbuf = (ctypes.c_uint8 * (max(n, 1) * 4 * nb))()
    pbuf = (ctypes.c_uint8 * (max(n, 1) * nb))()
    fbuf = (ctypes.c_uint8 * (4 * nb))()
    N.check(N.lib().zkl_matmul_prove(spec.fid, A.mtype, D.ptr(A.t), B.mtype, D.ptr(B.t), C.mtype,
                                     D.ptr(C.t), d0, d1, d2, state, rbuf, pbuf, fbuf, D.stream()))
    flat = D.decode(bytes(rbuf), spec, 4 * n)
    rounds = [tuple(flat[4 * j:4 * j + 4]) for j in range(n)]
    point = D.decode(bytes(pbuf), spec, n)
    finals = tuple(D.decode(bytes(fbuf), spec, 4))
    tr.state = state.raw[:64]
    log = getattr(tr, "log", None)
    if log is not None:  # the appends the reference makes (transcript.py:33-35)
        p = spec.modulus
        cneg = (-inverse_pow2(d1, p)) % p
        log.extend([(b"sumcheck/sum", 1), (b"sumcheck/shape", 3), (b"sumcheck/coeff", 1),
                    (b"sumcheck/factors", 3),
                    (b"sumcheck/coeff", (cneg.bit_length() + 7) >> 3 or 1),
                    (b"sumcheck/factors", 2)])
        log += [(b"sumcheck/eval", (e.bit_length() + 7) >> 3 or 1) for e in flat]
    return rounds, point, finals


def _records(pairs):
    """Transcript records (label, data) in the reference's framing
    (transcript.py:13-35): u16le |label| || label || u64le |data| || data."""
    out = bytearray()
    for label, data in pairs:
        if isinstance(data, int):
            data = data.to_bytes((data.bit_length() + 7) // 8 or 1, "little")
        out += len(label).to_bytes(2, "little") + label + len(data).to_bytes(8, "little") + data
    return bytes(out)


def matmul_sumcheck_batch(claims, tr, pre=None):
    """matmul_sumcheck for a sequence of claims on one transcript: claims is
    [(A, B, C, dims)], pre (optional) a list of [(label, data)] records
    appended to the transcript before each claim.  Returns the per-claim
    (rounds, point, final_values) -- the same proofs, and the same
    transcript, as

        for (A, B, C, dims), recs in zip(claims, pre):
            for label, data in recs: tr.append(label, data)
            matmul_sumcheck(A, B, C, dims, tr)

    With the native transcript the whole sequence is one C call
    (zkl_matmul_prove_batch): the next claim's challenge draws and matvecs are
    queued while the previous claim's last fold runs."""
    claims = list(claims)
    pre = list(pre) if pre is not None else [()] * len(claims)
    if len(pre) != len(claims):
        raise ValueError("one record list per claim")
    p = tr.modulus
    spec = D.spec_for(p)
    for A, B, C, dims in claims:
        d0, d1, d2 = dims
        D0, D1, D2 = 1 << d0, 1 << d1, 1 << d2
        if (A.rows, A.cols, B.rows, B.cols, C.rows, C.cols) != (D0, D1, D1, D2, D0, D2):
            raise ShapeMismatch("device operands do not match dims %r" % (dims,))
    if not (NATIVE_DRIVER and native_transcript(tr, spec)) or not claims:
        out = []
        for (A, B, C, dims), recs in zip(claims, pre):
            for label, data in recs:
                tr.append(label, data)
            out.append(matmul_sumcheck(A, B, C, dims, tr))
        return out
    k = len(claims)
    nb = spec.nbytes
    types = (ctypes.c_int * (3 * k))(*[M.mtype for c in claims for M in c[:3]])
    mats = (ctypes.c_void_p * (3 * k))(*[M.t.data_ptr() for c in claims for M in c[:3]])
    dims = (ctypes.c_int * (3 * k))(*[d for c in claims for d in c[3]])
    blobs = [_records(recs) for recs in pre]
    offs = [0]
    for b in blobs:
        offs.append(offs[-1] + len(b))
    blob = b"".join(blobs)
    pre_off = (ctypes.c_uint64 * (k + 1))(*offs)
    total = sum(sum(c[3]) for c in claims)
    state = ctypes.create_string_buffer(bytes(tr.state), 64)
    rbuf = (ctypes.c_uint8 * (max(total, 1) * 4 * nb))()
    pbuf = (ctypes.c_uint8 * (max(total, 1) * nb))()
    fbuf = (ctypes.c_uint8 * (4 * nb * k))()
    N.check(N.lib().zkl_matmul_prove_batch(spec.fid, k, types, mats, dims, blob or None,
                                           pre_off if blob else None, state, rbuf, pbuf, fbuf,
                                           D.stream()))
    flat = D.decode(bytes(rbuf), spec, 4 * total)
    pts = D.decode(bytes(pbuf), spec, total)
    fins = D.decode(bytes(fbuf), spec, 4 * k)
    tr.state = state.raw[:64]
    log = getattr(tr, "log", None)
    out = []
    o = 0
    for i, ((A, B, C, dims), recs) in enumerate(zip(claims, pre)):
        n = sum(dims)
        ev = flat[4 * o:4 * (o + n)]
        out.append(([tuple(ev[4 * j:4 * j + 4]) for j in range(n)], pts[o:o + n],
                    tuple(fins[4 * i:4 * i + 4])))
        if log is not None:
            for label, data in recs:
                ln = len(data) if not isinstance(data, int) else (data.bit_length() + 7) // 8 or 1
                log.append((label, ln))
            cneg = (-inverse_pow2(dims[1], p)) % p
            log.extend([(b"sumcheck/sum", 1), (b"sumcheck/shape", 3), (b"sumcheck/coeff", 1),
                        (b"sumcheck/factors", 3),
                        (b"sumcheck/coeff", (cneg.bit_length() + 7) >> 3 or 1),
                        (b"sumcheck/factors", 2)])
            log += [(b"sumcheck/eval", (e.bit_length() + 7) >> 3 or 1) for e in ev]
        o += n
    return out


def matmul_sumcheck(A, B, C, dims, tr):
    """The sumcheck of prove_matmul (gadgets.py:241-251), factored, on the GPU.

    A, B, C: DeviceMatrix of shapes 2^d0 x 2^d1, 2^d1 x 2^d2, 2^d0 x 2^d2.
    Starts by drawing r_u / r_v; returns (rounds, point, final_values) with
    rounds as evaluation tuples, identical to the reference's.
    """
    p = tr.modulus
    spec = D.spec_for(p)
    d0, d1, d2 = dims
    D0, D1, D2 = 1 << d0, 1 << d1, 1 << d2
    if (A.rows, A.cols, B.rows, B.cols, C.rows, C.cols) != (D0, D1, D1, D2, D0, D2):
        raise ShapeMismatch("device operands do not match dims %r" % (dims,))
    if NATIVE_DRIVER and native_transcript(tr, spec):
        return _matmul_native(A, B, C, dims, tr, spec)
    r_u = tr.challenge_vector(b"matmul/r_u", d0)
    r_v = tr.challenge_vector(b"matmul/r_v", d2)
    cneg = (-inverse_pow2(d1, p)) % p
    absorb_claim(tr, 0, [Term(1, (0, 1, 2)), Term(cneg, (0, 3))], 3, d0 + d1 + d2)
    E_v = D.eq_table(r_v, spec)

    # U phase
    bv = _matvec(B, E_v, False, spec)
    cv = _matvec(C, E_v, False, spec)
    abv = _matvec(A, bv, False, spec)
    h = _axpy(abv, cneg * pow(2, d1, p) % p, cv, D0, spec)
    if d0:
        E_u = D.eq_table(r_u, spec)
        rounds_u, pt_u, fin_u = run_rounds(spec, [E_u, h], d0, [(1, (0, 1))], 3, tr)
        e_hat = fin_u[0]
    else:
        rounds_u, pt_u, e_hat = [], [], 1

    # W phase
    E_ru = D.eq_table(pt_u, spec)
    a = _matvec(A, E_ru, True, spec)
    cu = _matvec(C, E_ru, True, spec)
    kappa = D.dot(cu, E_v, spec, D2)
    if d1:
        adds = [cneg * pow(2, d1 - j - 1, p) % p * kappa % p for j in range(d1)]
        rounds_w, pt_w, fin_w = run_rounds(spec, [a, bv], d1, [(1, (0, 1))], 3, tr,
                                           post_add=adds, post_mul=e_hat)
        alpha_s = fin_w[0]
    else:
        rounds_w, pt_w, alpha_s = [], [], D.read_scalar(a, spec)

    # V phase
    E_rw = D.eq_table(pt_w, spec)
    bw = _matvec(B, E_rw, True, spec)
    if d2:
        rounds_v, pt_v, fin_v = run_rounds(
            spec, [E_v, bw, cu], d2, [(alpha_s, (0, 1)), (cneg, (0, 2))], 3, tr,
            post_mul=e_hat)
        ev, bw_f, cu_f = fin_v
    else:
        rounds_v, pt_v = [], []
        ev, bw_f, cu_f = 1, D.read_scalar(bw, spec), D.read_scalar(cu, spec)
    finals = (e_hat * ev % p, alpha_s, bw_f, cu_f)
    return rounds_u + rounds_w + rounds_v, pt_u + pt_w + pt_v, finals


def replicated_tables(A, B, C, dims, r_u, r_v, spec):
    """The reference's four zkMat tables (gadgets.py:210-227) materialised on
    the device: [eq(r_u,u) eq(r_v,v), A(u,w), B(w,v), C(u,v)] over the index
    u || w || v (MSB first), 2^(d0+d1+d2) field elements each."""
    d0, d1, d2 = dims
    D0, D1, D2 = 1 << d0, 1 << d1, 1 << d2
    W = spec.nbytes // 8
    uv = D.eq_table(list(r_u) + list(r_v), spec)  # eq(r_u,u) eq(r_v,v) over u || v
    a = A.as_field_vector(spec).view(D0, D1, 1, W)
    b = B.as_field_vector(spec).view(1, D1, D2, W)
    c = C.as_field_vector(spec).view(D0, 1, D2, W)
    shape = (D0, D1, D2, W)
    return [uv.view(D0, 1, D2, W).expand(shape).reshape(-1, W),
            a.expand(shape).reshape(-1, W), b.expand(shape).reshape(-1, W),
            c.expand(shape).reshape(-1, W)]


def matmul_sumcheck_replicated(A, B, C, dims, tr):
    """The reference's own zkMat sumcheck form (gadgets.py:241-251): the four
    replicated tables materialised and proven by the dense fused round/fold
    engine over d0+d1+d2 rounds.  Same transcript traffic and outputs as
    matmul_sumcheck (the factored prover); it exists for the like-for-like
    scaling sweep (BASELINE config 5) and as a cross-check of the factored
    path at sizes the CPU oracle cannot reach."""
    p = tr.modulus
    spec = D.spec_for(p)
    d0, d1, d2 = dims
    r_u = tr.challenge_vector(b"matmul/r_u", d0)
    r_v = tr.challenge_vector(b"matmul/r_v", d2)
    cneg = (-inverse_pow2(d1, p)) % p
    n = d0 + d1 + d2
    terms = [(1, (0, 1, 2)), (cneg, (0, 3))]
    g = shard.active()
    if shard.wants(n) and (1 << d2) >= g.world and native_transcript(tr, spec):
        # multi-GPU: the low index bits are v's, so this rank's shard of the
        # four tables is the replicated claim over the columns v = v' G + rank
        tables = replicated_tables_shard(A, B, C, dims, r_u, r_v, spec, g.rank, g.world)
        absorb_claim(tr, 0, [Term(c, f) for c, f in terms], 3, n)
        return shard.run_rounds_sharded(spec, tables, n, terms, 3, tr)
    tables = replicated_tables(A, B, C, dims, r_u, r_v, spec)
    absorb_claim(tr, 0, [Term(1, (0, 1, 2)), Term(cneg, (0, 3))], 3, n)
    return run_rounds(spec, tables, n, terms, 3, tr)


def replicated_tables_shard(A, B, C, dims, r_u, r_v, spec, rank, world):
    """Rank `rank`'s cyclic shard of replicated_tables: global index
    u || w || v with v = v' world + rank, i.e. the replicated claim of the
    column slices B[:, rank::world], C[:, rank::world] and the eq weights
    eq(r_u, u) eq(r_v, v' world + rank)."""
    d0, d1, d2 = dims
    D0, D1, D2 = 1 << d0, 1 << d1, (1 << d2) // world
    W = spec.nbytes // 8
    uv = shard.eq_shard(list(r_u) + list(r_v), spec, rank, world)  # over u || v'
    a = A.as_field_vector(spec).view(D0, D1, 1, W)
    def cols(M, rows):
        if M.mtype == N.MT_FIELD:
            t = M.t.view(rows, 1 << d2, W)[:, rank::world].reshape(-1, W).contiguous()
            return DeviceMatrix(t, rows, D2, N.MT_FIELD, spec).as_field_vector(spec)
        t = M.t.view(rows, 1 << d2)[:, rank::world].contiguous()
        return DeviceMatrix.from_int_tensor(t).as_field_vector(spec)

    b, c = cols(B, D1), cols(C, D0)
    b = b.view(1, D1, D2, W)
    c = c.view(D0, 1, D2, W)
    shape = (D0, D1, D2, W)
    return [uv.view(D0, 1, D2, W).expand(shape).reshape(-1, W),
            a.expand(shape).reshape(-1, W), b.expand(shape).reshape(-1, W),
            c.expand(shape).reshape(-1, W)]


def prove_matmul(a, b, c, key, tr, rng):
    """Drop-in for zklora.gadgets.prove_matmul (gadgets.py:230-265)."""
    p = tr.modulus
    d0, d1 = a.ref.row_vars, a.ref.col_vars
    d1b, d2 = b.ref.row_vars, b.ref.col_vars
    if d1 != d1b or (c.ref.row_vars, c.ref.col_vars) != (d0, d2):
        raise ShapeMismatch(
            "matmul shapes (%d,%d)x(%d,%d)->(%d,%d) do not conform"
            % (d0, d1, d1b, d2, c.ref.row_vars, c.ref.col_vars))
    _absorb_operands(tr, b"matmul", [a.ref, b.ref, c.ref], key.group)
    spec = D.spec_for(p)
    D0, D1, D2 = 1 << d0, 1 << d1, 1 << d2
    A = _device_matrix(a, D0, D1, spec)
    B = _device_matrix(b, D1, D2, spec)
    C = _device_matrix(c, D0, D2, spec)
    rounds, point, finals = matmul_sumcheck(A, B, C, (d0, d1, d2), tr)
    RP = SC_TYPES["RoundPolynomial"]
    sc_proof = SC_TYPES["SumcheckProof"]([RP(e) for e in rounds], tuple(finals))
    rho_u, rho_w, rho_v = point[:d0], point[d0:d0 + d1], point[d0 + d1:]

    def maybe_open(pt, opening_point, value):
        if pt.ref.kind != "committed":
            return None
        return _open_tables(key, [pt], opening_point, tr, rng, values=[value])

    return TYPES["MatmulProof"](
        dims=(d0, d1, d2),
        sumcheck=sc_proof,
        a_opening=maybe_open(a, rho_u + rho_w, finals[1]),
        b_opening=maybe_open(b, rho_w + rho_v, finals[2]),
        c_opening=maybe_open(c, rho_u + rho_v, finals[3]),
    )


def prove_matadd(a, b, c, sign, key, tr, rng):
    """Drop-in for zklora.gadgets.prove_matadd (gadgets.py:322-336): c = a +
    sign*b checked at one random point, i.e. a batch opening of the committed
    operands (device MLE evaluations for DeviceMatrix operands)."""
    shape = (a.ref.row_vars, a.ref.col_vars)
    if (b.ref.row_vars, b.ref.col_vars) != shape or (c.ref.row_vars, c.ref.col_vars) != shape:
        raise ShapeMismatch("matadd operands must share a shape")
    if sign not in (1, -1):
        raise ValueError("sign must be +1 or -1")
    _absorb_operands(tr, b"matadd", [a.ref, b.ref, c.ref], key.group)
    tr.append(b"matadd/sign", sign % tr.modulus)
    point = tr.challenge_vector(b"matadd/point", a.ref.num_vars)
    committed = [t for t in (a, b, c) if t.ref.kind == "committed"]
    opening = _open_tables(key, committed, point, tr, rng) if committed else None
    return TYPES["MataddProof"](sign=sign, shape=shape, opening=opening)


def _consumable(M, spec):
    """A fresh field copy of a DeviceMatrix that a sumcheck may fold in place
    (integer matrices are lifted straight into it)."""
    if M.mtype == N.MT_FIELD:
        return M.t.clone()
    return D.lift(M.t.reshape(-1), spec)


EQ_FACTORED_MIN_VARS = 20  # below this the dense engine's eq table costs nothing
EQ_TILE_LOG = 16


def _eq_factored_prod3(spec, tr, r, ta, tb, n):
    """The elementprod claim sum_i eq(r, i) A(i) B(i) (gadgets.py:396-405)
    without materialising eq(r, .): the first n - 16 rounds run on the
    eq-factored tiled evaluator of the logUp engine (eq = C_j l_j(x)
    eq_hi(k) eq_lo(t); term coefficients (1, 0, 0, 0, 0) reduce its claim to
    E A S; 6 Montgomery products per pair in round 0 and 10 after, against 7
    and 13 with the table), then the last 16 rounds over E bound at the point,
    A and B.  Same rounds, point and finals as the dense claim; None when the
    native engine declines (stepwise mode under profilers)."""
    if not native_transcript(tr, spec):
        return None
    tile_log = EQ_TILE_LOG
    r1 = n - tile_log
    nt = 1 << tile_log
    E = D.empty(spec, nt)
    side = D.empty(spec, nt).zero_()  # the logUp table-side columns: unused (coefficients 0)
    nb = spec.nbytes
    state = ctypes.create_string_buffer(bytes(tr.state), 64)
    rbuf = (ctypes.c_uint8 * (r1 * 4 * nb))()
    pbuf = (ctypes.c_uint8 * (r1 * nb))()
    ptrs = (ctypes.c_void_p * 6)(*[t.data_ptr() for t in (E, ta, tb, side, side, side)])
    coeffs = D.scalars_bytes([1, 0, 0, 0, 0], spec)
    rc = N.lib().zkl_logup_tiled_rounds(spec.fid, ptrs, tile_log, n, r1,
                                        D.scalars_bytes(list(r), spec), coeffs, 0, state, rbuf,
                                        pbuf, D.stream())
    if rc == N.ZKL_ERR_UNSUPPORTED:
        return None
    N.check(rc)
    flat = D.decode(bytes(rbuf), spec, 4 * r1)
    rounds = [tuple(flat[4 * j:4 * j + 4]) for j in range(r1)]
    point = D.decode(bytes(pbuf), spec, r1)
    tr.state = state.raw[:64]
    log = getattr(tr, "log", None)
    if log is not None:
        log.extend((b"sumcheck/eval", (e.bit_length() + 7) // 8 or 1) for e in flat)
    r2, p2, finals = run_rounds(spec, [E, ta[:nt], tb[:nt]], tile_log, [(1, (0, 1, 2))], 3, tr)
    return rounds + r2, point + p2, finals


def prove_elementprod(a, b, c, key, tr, rng):
    """Drop-in for zklora.gadgets.prove_elementprod (gadgets.py:383-410)."""
    p = tr.modulus
    shape = (a.ref.row_vars, a.ref.col_vars)
    if (b.ref.row_vars, b.ref.col_vars) != shape or (c.ref.row_vars, c.ref.col_vars) != shape:
        raise ShapeMismatch("elementprod operands must share a shape")
    if c.ref.kind != "committed":
        raise ValueError("elementprod output must be committed")
    _absorb_operands(tr, b"elementprod", [a.ref, b.ref, c.ref], key.group)
    n = a.ref.num_vars
    r = tr.challenge_vector(b"elementprod/r", n)
    c_opening = _open_tables(key, [c], r, tr, rng)
    claimed = c_opening.values[0]
    spec = D.spec_for(p)
    rows, cols = 1 << shape[0], 1 << shape[1]
    term = Term(1, (0, 1, 2))
    if shard.wants(n) and native_transcript(tr, spec):
        # multi-GPU: this rank's cyclic shard of eq(r, .), A and B (shard.py)
        g = shard.active()
        absorb_claim(tr, claimed, [term], 3, n)
        loc = [shard.eq_shard(r, spec, g.rank, g.world),
               _shard_matrix(_device_matrix(a, rows, cols, spec), spec, g),
               _shard_matrix(_device_matrix(b, rows, cols, spec), spec, g)]
        rounds, point, finals = shard.run_rounds_sharded(spec, loc, n, [(1, (0, 1, 2))], 3, tr)
        return _elementprod_proof(key, tr, rng, a, b, shape, c_opening, rounds, point, finals)
    ta = _consumable(_device_matrix(a, rows, cols, spec), spec)
    tb = _consumable(_device_matrix(b, rows, cols, spec), spec)
    absorb_claim(tr, claimed, [term], 3, n)
    got = _eq_factored_prod3(spec, tr, r, ta, tb, n) if n >= EQ_FACTORED_MIN_VARS else None
    if got is not None:
        rounds, point, finals = got
    elif n:
        rounds, point, finals = run_rounds(spec, [D.eq_table(r, spec), ta, tb], n,
                                           [(1, (0, 1, 2))], 3, tr)
    else:
        rounds, point = [], []
        finals = [1, D.read_scalar(ta, spec), D.read_scalar(tb, spec)]
    return _elementprod_proof(key, tr, rng, a, b, shape, c_opening, rounds, point, finals)


def _shard_matrix(M, spec, g):
    """This rank's cyclic shard (entries i*G + rank of the row-major matrix)
    as a fresh field vector: integer matrices are sliced first, then lifted."""
    if M.mtype == N.MT_FIELD:
        return shard.shard_of(M.t, spec, g.rank, g.world)
    return D.lift(M.t.reshape(-1)[g.rank::g.world].contiguous(), spec)


def _elementprod_proof(key, tr, rng, a, b, shape, c_opening, rounds, point, finals):
    RP = SC_TYPES["RoundPolynomial"]
    sc_proof = SC_TYPES["SumcheckProof"]([RP(e) for e in rounds], tuple(finals))
    committed = [t for t in (a, b) if t.ref.kind == "committed"]
    vals = [finals[1] if t is a else finals[2] for t in committed]
    ab_opening = _open_tables(key, committed, point, tr, rng, values=vals) if committed else None
    return TYPES["ElementprodProof"](shape=shape, c_opening=c_opening, sumcheck=sc_proof,
                                     ab_opening=ab_opening)


# ---------------------------------------------------------------------------
# pair-table lookups (gadgets.py:659-688)
def _combine_commitments(key, commitments, coefficients):
    """commit.combine_commitments, or the stub's (same num_vars) for StubKey."""
    if getattr(key, "is_stub", False):
        from .commit_stub import combine_commitments

        return combine_commitments(key.group, commitments, coefficients)
    import zklora.commit as zc

    return zc.combine_commitments(key.group, commitments, coefficients)


def _int_column(entries):
    """A device integer column (torch int16/32/64 CUDA tensor) or None."""
    return entries if torch.is_tensor(entries) and entries.is_cuda else None


def prove_pair_lookup(label, x, y, pair_table, key, tr, rng):
    """Mirror of zklora.gadgets._prove_pair_lookup (gadgets.py:679-688).

    Same transcript traffic: x / y digests, alpha, then prove_lookup on the
    compressed secret x + alpha*y against the compressed table
    (tables.py:131-140).  When x / y carry device integer matrices and the
    pair table's columns are device integer tensors, the compression,
    multiplicities and the whole lookup stay on the GPU (DeviceVector
    entries); otherwise the reference's list semantics apply.
    """
    from .lookup import (LookupTable, SecretVector, compute_multiplicities,
                         multiplicities_indexed, multiplicities_pair, prove_lookup)

    p = tr.modulus
    tr.append(label + b"/x", x.ref.digest(key.group))
    tr.append(label + b"/y", y.ref.digest(key.group))
    alpha = tr.challenge(label + b"/alpha")
    spec = D.spec_for(p)
    xd, yd = getattr(x, "device", None), getattr(y, "device", None)
    tx, ty = _int_column(pair_table.x.entries), _int_column(pair_table.y.entries)
    secret_com = _combine_commitments(key, [x.ref.commitment, y.ref.commitment], [1, alpha])
    table_com = _combine_commitments(key, [pair_table.x.commitment, pair_table.y.commitment],
                                     [1, alpha])
    rows = 1 << ((x.ref.num_vars + 1) // 2)
    bx = list(x.blinding) if x.blinding else [0] * rows
    by = list(y.blinding) if y.blinding else [0] * rows
    if any(by):
        blinding = tuple((a + alpha * b) % p for a, b in zip(bx, by))
    else:  # (the stub / unblinded case: skip 2^13 bigint products per lookup)
        blinding = tuple(a % p for a in bx)
    if (xd is not None and yd is not None and xd.mtype != N.MT_FIELD
            and yd.mtype != N.MT_FIELD and tx is not None and ty is not None):
        secret = SecretVector(D.PairColumn(xd.t, yd.t, alpha, spec), secret_com, blinding)
        table = LookupTable(D.pair_combine(tx, ty, alpha, spec), table_com,
                            pair_table.name + "+a*y")
    else:
        xs, ys = x.flat(), y.flat()
        secret = SecretVector(tuple((a + alpha * b) % p for a, b in zip(xs, ys)), secret_com,
                              blinding)
        table = LookupTable(tuple((a + alpha * b) % p for a, b in
                                  zip(pair_table.x.entries, pair_table.y.entries)),
                            table_com, pair_table.name + "+a*y")
    if isinstance(secret.entries, D.DeviceVector):
        got = None
        if xd is not None and yd is not None and tx is not None and ty is not None:
            got = multiplicities_pair(secret.entries, table, xd.t, yd.t, tx, ty)
        counts, index = got if got is not None else multiplicities_indexed(secret.entries, table)
        return prove_lookup(secret, counts, table, key, tr, rng, secret_index=index)
    counts = compute_multiplicities(secret.entries, table)
    return prove_lookup(secret, counts, table, key, tr, rng)
