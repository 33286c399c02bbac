"""LoRA transformer-block proof schedule (BASELINE configs 4/5, "LoRA-block
proof seconds"), composed from this backend's gadget provers.

The reference cannot express these blocks (SURVEY.md sec. 7 hard part 6:
pow-2 dims only, single head, LayerNorm, LoRA on W_V only), so the schedule is
a new composition of the reference's gadget API, every instance proven by the
drop-ins here on one sequential Fiat-Shamir transcript:

  prove_matmul       gadgets.py:230-265   every fwd / bwd / LoRA-gradient matmul,
                                          row sums and broadcasts (ones vectors)
  prove_matadd       gadgets.py:322-336   residual adds, LoRA sums, softmax shift,
                                          gradient sums, the LoRA update
  prove_elementprod  gadgets.py:383-410   RMSNorm square / scaling, attention
                                          constant, softmax normalisation, SwiGLU
                                          gate products and their gradients
  prove_rescale      gadgets.py:600-622   every wide -> int16 narrowing (any
                                          divisor of zeta) incl. the update step
  prove_swiglu       gadgets.py:761-782   SiLU / SiLU' of the gate
  prove_rsqrt        gadgets.py:842-847   RMSNorm 1/sqrt(mean square)
  _prove_pair_lookup gadgets.py:679-688   softmax: row-shifted exp, one 2^16 segment

It follows the reference's own model graph where the reference has one:
RMSNorm's mean square is the reference layernorm's (model.py:640-661: narrow by
s = 2^ceil(k/2), square, row-sum by a ones matmul, narrow by gamma*d/s^2,
rsqrt lookup, broadcast by a ones matmul); the score constant is an elementprod
with a public constant (model.py:716-717); the softmax backward is
model.py:785-791; the LoRA update is model.py:823-836 (rescale by 1/eta, then
matadd).  Two values are computed, not proven: the softmax row maximum (any
shift gives the same softmax; the lookup proves the shifted scores lie in the
exp table's domain) and the row-sum reciprocal (the reference proves softmax
normalisation only through its per-row gadget, gadgets.py:930-1036).

Fixed point.  Every tensor is int16 (int32 / int64 for table outputs and wide
products) at a power-of-two scale 2^e.  A rescale by divisor 2^k (k <= log2
zeta, gadgets.py:566) takes a wide product at 2^(ea+eb) to 2^(ea+eb-k).  The
per-tensor exponents below keep every quotient inside quant_range (|x| < 8 at
2^12), because the reference prover raises RangeViolation otherwise
(gadgets.py:575) and a clamped quotient breaks the identity its verifier checks
(gadgets.py:644, 803).  The witness pass raises the same way; nothing is
clipped.  gamma_fp = zeta = 2^g (g = 12 at LLaMA shape):

  X, xn, p, out, x1, dY and activation grads       2^g
  W_q, W_k, W_v; q, k, v; o; LoRA A, hidden x A     2^(g-1)
  LoRA B (one above its W: B_q/k/v 2^g, B_o 2^(g+1))
  score constant 1/sqrt(d_head); qc                2^(g-1); 2^(g-2)
  scores z, shifted scores (exp table base 4)      2^(g-2)   (|z| < 32)
  W_g; SiLU / SiLU' tables (gamma/2, act 16)       2^(g-1)
  W_u; up                                          2^(g-3)
  gate * up, down projection                       2^(g-4)   (|.| < 128)

Witnesses are seeded synthetic tensors: X ~ N(0,1), weights ~ N(0,0.02)
quantised at their exponent above (W_q carries no scale: the score constant
is proven), upstream gradient dY ~ N(0,1e-3) (a per-token gradient of a mean
loss; BASELINE cfg4 leaves it open), exact int64 products via float64 GEMMs
(|partial sums| < 2^53).  Dimensions that are not powers of two are
zero-padded (quantize.py:176-183); RMSNorm then averages over the padded row
(the divisor must be a power of two), i.e. a gain of sqrt(d_pad / d).
Commitments use the deterministic stub (commit_stub.py).
"""

import math
import time
from collections import defaultdict
from dataclasses import dataclass

import numpy as np
import torch

from . import tables as TBL
from .commit_stub import StubCommitment, StubKey, attach
from .device import igemm16
from .gadgets import (DeviceMatrix, ProverTensor, TensorRef, prove_elementprod, prove_matadd,
                      prove_matmul, prove_pair_lookup)
from .nonlinear import (RangeViolation, TableSet, device_pair_table, device_range_table,
                        prove_rescale, prove_rsqrt, prove_swiglu, rescale_witness_device)


@dataclass(frozen=True)
class BlockShape:
    name: str
    seq: int
    hidden: int
    heads: int
    head_dim: int
    ffn: int
    rank: int
    lora: tuple  # projections with LoRA adapters, subset of "qkvo"


LLAMA2_7B = BlockShape("llama2-7b", 2048, 4096, 32, 128, 11008, 8, ("q", "v"))
LLAMA2_13B = BlockShape("llama2-13b", 2048, 5120, 40, 128, 13824, 16, ("q", "k", "v", "o"))


@dataclass(frozen=True)
class FixedPoint:
    """QuantParams fields the block reads (quantize.py): gamma_fp = zeta =
    2^12, act_bound 8, RMSNorm eps 1e-5; the softmax exp table is the
    reference's exp segment with base `exp_base` (tables.py:56-62; scores at
    gamma/exp_base); the SiLU tables are built at gamma >> act_shift (inputs
    |x| < act_bound << act_shift); the LoRA learning rate is 1/eta_div
    (model.py:104-106)."""

    gamma_fp: int = 1 << 12
    zeta: int = 1 << 12
    act_bound: int = 8
    exp_n: int = 1 << 16
    eps: float = 1e-5
    exp_base: int = 4
    act_shift: int = 1
    eta_div: int = 256

    @property
    def qmin(self):
        return -self.act_bound * self.gamma_fp

    @property
    def qmax(self):
        return self.act_bound * self.gamma_fp - 1

    @property
    def g(self):
        return self.gamma_fp.bit_length() - 1


FP = FixedPoint()


def _p2(n):
    return 1 << (n - 1).bit_length()


def _log2(n):
    return (n - 1).bit_length()


def block_tables(spec, fp=FP):
    """The TableSet of the block (tables.py:217-238 fields) on the device."""
    g, a = fp.gamma_fp, fp.act_bound
    ga, aa = g >> fp.act_shift, a << fp.act_shift

    def com(n):
        return StubCommitment(_log2(n))

    lo, n = TBL.quant_range(g, a)
    quant = device_range_table(lo, n, spec, com(n), "quant_range")
    lo, n = TBL.residue_range(fp.zeta)
    resid = device_range_table(lo, n, spec, com(n), "residue_range")

    def pair(cols, name):
        n = len(cols[0])
        return device_pair_table(*cols, com(n), com(n), name)

    exp = TBL.exp_segment_entries(g, (fp.exp_base, fp.exp_n), 1)
    return TableSet(fp, fp.eps, spec.modulus, b"", (pair(exp, "exp0"),),
                    pair(TBL.silu_entries(ga, aa), "silu"),
                    pair(TBL.silu_deriv_entries(ga, aa), "silu_deriv"),
                    pair(TBL.rsqrt_entries(g, a, fp.eps), "rsqrt"), quant, resid)


def block_luts(tables):
    """Witness-side table outputs (int32 columns) keyed by name, with the
    first input of each table."""
    return {"silu": tables.silu.y.entries, "silu_deriv": tables.silu_deriv.y.entries,
            "rsqrt": tables.rsqrt.y.entries, "exp": tables.exp_segments[0].y.entries,
            "act_x0": int(tables.silu.x.entries[0])}


# ---------------------------------------------------------------------------
# fixed-point witness arithmetic (device, untimed)
def _q16(rng, shape, std, rows, cols, scale, device):
    """round_half_away(N(0,std) * scale) as int16 (out of range raises),
    zero-padded to (rows, cols)."""
    a = rng.standard_normal(shape) * std * scale
    a = np.sign(a) * np.floor(np.abs(a) + 0.5)
    if a.size and (a.min() < -32768 or a.max() > 32767):
        raise RangeViolation("synthetic tensor outside int16 at scale %g" % scale)
    t = torch.zeros((rows, cols), dtype=torch.int16)
    t[: shape[0], : shape[1]] = torch.from_numpy(a.astype(np.int16))
    return t.to(device)


def _mm(a, b):
    """Exact int64 a @ b of integer matrices: int16 x int16 on the GPU through
    the byte-sliced tensor-core GEMM (device.igemm16); the ones-vector row sums
    and broadcasts (int32 / int64 operands) and CPU tensors through a float64
    GEMM, exact because every partial sum stays below 2^53 (checked)."""
    if a.is_cuda and a.dtype == torch.int16 and b.dtype == torch.int16:
        return igemm16(a, b)
    out = torch.matmul(a.double(), b.double())
    assert float(out.abs().max()) < 2.0 ** 52 if out.numel() else True
    return out.round_().long()


def _divmod(wide, divisor, fp):
    """centered_divmod (quantize.py:101-104) by `divisor` with the quant_range
    check of rescale_witness (gadgets.py:565-580): (q int16, r * zeta/divisor
    int16).  On the GPU one fused pass (nonlinear.rescale_witness_device); the
    torch form is the CPU path the golden generator drives the reference with."""
    if wide.is_cuda:
        return rescale_witness_device(wide, divisor, fp)
    if divisor <= 0 or fp.zeta % divisor:
        raise ValueError("divisor must divide zeta")
    q = torch.div(wide + divisor // 2, divisor, rounding_mode="floor")
    bad = (q < fp.qmin) | (q > fp.qmax)
    if bool(bad.any()):
        raise RangeViolation("rescale quotient %d outside table domain (%d entries)"
                             % (int(q[bad].reshape(-1)[0]), int(bad.sum())))
    r = (wide - divisor * q) * (fp.zeta // divisor)
    return q.to(torch.int16), r.to(torch.int16)


def _add(a, b, sign, dtype=torch.int16):
    """a + sign*b, the matadd witness; raises if it leaves `dtype`."""
    c = a.long() + sign * b.long()
    info = torch.iinfo(dtype)
    if c.numel() and (int(c.min()) < info.min or int(c.max()) > info.max):
        raise RangeViolation("matadd output outside %s" % dtype)
    return c.to(dtype)


def _lut(table_y, x, x0):
    return table_y[(x.long() - x0)]


class _Rng:
    def vector(self, n):
        return [0] * n


class BlockProver:
    """One sequential transcript over the whole block; records per-gadget
    counts, rounds, field elements and seconds.

    on_proof(kind, refs, proof), when given, is called after every gadget with
    the operand TensorRefs and the proof (the verifier-in-the-loop harness,
    harness/refverify.py, runs the reference's verifier there)."""

    def __init__(self, tr, tables, key=None, timing=True, on_proof=None):
        self.tr, self.tables = tr, tables
        self.timing = timing  # per-gadget synchronised spans (off: the host runs ahead)
        self.fp = tables.params
        self.luts = block_luts(tables)
        self.key = key or StubKey()
        self.on_proof = on_proof
        self.stats = defaultdict(lambda: [0, 0, 0, 0.0])  # count, rounds, elems, seconds
        self.log = []  # [kind, rounds of each sumcheck] per gadget, in proof order
        self.seconds = []  # per gadget, same order as log

    def pt(self, t):
        rv, cv = _log2(t.shape[0]), _log2(t.shape[1])
        dm = DeviceMatrix.from_int_tensor(t)
        ref = TensorRef("committed", rv, cv, commitment=attach(StubCommitment(rv + cv), dm))
        return ProverTensor(None, ref, (), device=dm)

    def _run(self, kind, fn, *args):
        if not self.timing:
            out = fn(*args)
            self.stats[kind][0] += 1
            self.seconds.append(0.0)
            return out
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*args)
        torch.cuda.synchronize()
        s = self.stats[kind]
        dt = time.perf_counter() - t0
        s[0] += 1
        s[3] += dt
        self.seconds.append(dt)
        return out

    def _count(self, kind, rounds, elems):
        s = self.stats[kind]
        s[1] += rounds
        s[2] += elems

    def _done(self, kind, ops, proof, extra=None):
        if self.on_proof is not None:
            self.on_proof(kind, [o.ref for o in ops], proof, extra)

    def matmul(self, a, b, c):
        ops = [self.pt(a), self.pt(b), self.pt(c)]
        pr = self._run("matmul", prove_matmul, *ops, self.key, self.tr, _Rng())
        n = sum(pr.dims)
        self._count("matmul", n, 4 << n)
        self.log.append(["matmul", len(pr.sumcheck.rounds)])
        self._done("matmul", ops, pr)

    def matadd(self, a, b, c, sign):
        ops = [self.pt(a), self.pt(b), self.pt(c)]
        pr = self._run("matadd", prove_matadd, *ops, sign, self.key, self.tr, _Rng())
        self.log.append(["matadd"])
        self._done("matadd", ops, pr)

    def eprod(self, a, b, c):
        ops = [self.pt(a), self.pt(b), self.pt(c)]
        pr = self._run("elementprod", prove_elementprod, *ops, self.key, self.tr, _Rng())
        n = sum(pr.shape)
        self._count("elementprod", n, 3 << n)
        self.log.append(["elementprod", len(pr.sumcheck.rounds)])
        self._done("elementprod", ops, pr)

    def _lookups(self, kind, lps):
        self.log.append([kind] + [len(lp.sumcheck.rounds) for lp in lps])
        for lp in lps:
            n = len(lp.sumcheck.rounds)
            self._count(kind, n, 7 << n)

    def rescale(self, wide, divisor):
        q, r = _divmod(wide, divisor, self.fp)
        self.rescale_w(wide, q, r, divisor)
        return q

    def rescale_w(self, wide, q, r, divisor):
        ops = [self.pt(wide), self.pt(q), self.pt(r)]
        pr = self._run("rescale", prove_rescale, *ops, divisor, self.tables, self.key, self.tr,
                       _Rng())
        self._lookups("rescale", (pr.quant_lookup, pr.resid_lookup))
        self._done("rescale", ops, pr)

    def swiglu(self, wide, mode):
        q, r = _divmod(wide, self.fp.zeta, self.fp)
        table = self.luts["silu" if mode == "phi" else "silu_deriv"]
        out = _lut(table, q, self.luts["act_x0"]).to(torch.int16)
        self.swiglu_w(wide, out, q, r, mode)
        return out

    def swiglu_w(self, wide, out, q, r, mode):
        ops = [self.pt(wide), self.pt(out), self.pt(q), self.pt(r)]
        pr = self._run("swiglu", prove_swiglu, *ops, mode, self.tables, self.key, self.tr,
                       _Rng())
        self._lookups("swiglu", (pr.activation_lookup, pr.resid_lookup))
        self._done("swiglu", ops[:2], pr)

    def rsqrt(self, v, u):
        ops = [self.pt(v), self.pt(u)]
        pr = self._run("rsqrt", prove_rsqrt, *ops, self.tables, self.key, self.tr, _Rng())
        self._lookups("rsqrt", (pr.lookup,))
        self._done("rsqrt", ops, pr)

    def exp_lookup(self, v, e):
        ops = [self.pt(v), self.pt(e)]
        pr = self._run("softmax_exp", prove_pair_lookup, b"softmax/exp0", *ops,
                       self.tables.exp_segments[0], self.key, self.tr, _Rng())
        self._lookups("softmax_exp", (pr,))
        self._done("softmax_exp", ops, pr)


class WitnessRecorder:
    """The witness pass of a block: runs prove_block's schedule computing every
    gadget's witness (narrowed quotients, residues, table outputs) and records
    the gadget calls with their operands, proving nothing.  The reference's
    gadget provers take their witnesses as inputs (prove_rescale(wide, narrow,
    resid, ...), prove_swiglu(wide, out, narrow, resid, ...)), so
    replay(BlockProver) proves exactly what the interleaved schedule proves,
    with the witness computed before the timed region."""

    def __init__(self, tables):
        self.fp = tables.params
        self.luts = block_luts(tables)
        self.calls = []

    def matmul(self, a, b, c):
        self.calls.append(("matmul", a, b, c))

    def matadd(self, a, b, c, sign):
        self.calls.append(("matadd", a, b, c, sign))

    def eprod(self, a, b, c):
        self.calls.append(("eprod", a, b, c))

    def rescale(self, wide, divisor):
        q, r = _divmod(wide, divisor, self.fp)
        self.calls.append(("rescale_w", wide, q, r, divisor))
        return q

    def swiglu(self, wide, mode):
        q, r = _divmod(wide, self.fp.zeta, self.fp)
        table = self.luts["silu" if mode == "phi" else "silu_deriv"]
        out = _lut(table, q, self.luts["act_x0"]).to(torch.int16)
        self.calls.append(("swiglu_w", wide, out, q, r, mode))
        return out

    def rsqrt(self, v, u):
        self.calls.append(("rsqrt", v, u))

    def exp_lookup(self, v, e):
        self.calls.append(("exp_lookup", v, e))

    def replay(self, P):
        """Prove the recorded gadgets in order through P (a BlockProver)."""
        for name, *args in self.calls:
            getattr(P, name)(*args)
        return P


# ---------------------------------------------------------------------------
class BlockWitness:
    """Seeded weights and input of one block, padded to powers of two, each
    quantised at its exponent (module docstring)."""

    def __init__(self, shape, seed=0, fp=FP, device="cuda", wstd=0.02, dy_std=1e-3):
        self.shape = shape
        g = np.random.Generator(np.random.PCG64(seed))
        S, Dm, F, R = shape.seq, shape.hidden, shape.ffn, shape.rank
        Dp, Fp = _p2(Dm), _p2(F)
        self.Dp, self.Fp = Dp, Fp
        e = fp.g

        def q(sh, std, rows, cols, exp):
            return _q16(g, sh, std, rows, cols, float(2 ** exp), device)

        self.X = q((S, Dm), 1.0, S, Dp, e)
        self.W = {p: q((Dm, Dm), wstd, Dp, Dp, e - 1 if p in "qkv" else e) for p in "qkvo"}
        self.Wg = q((Dm, F), wstd, Dp, Fp, e - 1)
        self.Wu = q((Dm, F), wstd, Dp, Fp, e - 3)
        self.Wd = q((F, Dm), wstd, Fp, Dp, e)
        # LoRA: A at 2^(g-1) (the hidden x A stays in range at 13B), B one
        # exponent above its W so that (x A) B lands on x W's exponent
        self.eW = {p: e - 1 if p in "qkv" else e for p in "qkvo"}
        self.eA = e - 1
        self.eB = {p: self.eW[p] + 1 for p in shape.lora}
        self.A = {p: q((Dm, R), wstd, Dp, R, self.eA) for p in shape.lora}
        self.B = {p: q((R, Dm), wstd, R, Dp, self.eB[p]) for p in shape.lora}
        self.dY = q((S, Dm), dy_std, S, Dp, e)
        # public constants: the score scale 1/sqrt(d_head) at 2^(g-1)
        # (model.py:716 multiplies q by round(gamma/sqrt(d)))
        c = int(math.floor(2 ** (e - 1) / math.sqrt(shape.head_dim) + 0.5))
        self.Cq = torch.zeros((S, Dp), dtype=torch.int16, device=device)
        self.Cq[:, :Dm] = c


def _t(x):
    return x.t().contiguous()


def _heads(x, H, dh):
    return [x[:, h * dh:(h + 1) * dh].contiguous() for h in range(H)]


def _stack_rows(mats, rows):
    """Stack (S x C) matrices vertically and zero-pad to `rows` rows."""
    out = torch.zeros((rows, mats[0].shape[1]), dtype=mats[0].dtype, device=mats[0].device)
    torch.cat(mats, out=out[: sum(m.shape[0] for m in mats)])
    return out


def _ones(rows, cols, valid, dev, dim):
    """Public ones vector (rows x cols) with zeros past `valid` along dim."""
    t = torch.zeros((rows, cols), dtype=torch.int16, device=dev)
    if dim == 0:
        t[:valid] = 1
    else:
        t[:, :valid] = 1
    return t


def prove_block(w, P):
    """Prove one LoRA fine-tuning step of one transformer block (forward,
    backward, LoRA gradients, LoRA update) through the gadget prover P
    (BlockProver, WitnessRecorder, or a stand-in with the same methods that
    drives the reference's gadgets for parity goldens).  Returns P.

    Exponents (log2 scales, g = log2 gamma) are noted as @e; a rescale by
    divisor 2^k maps a wide product @e to @(e-k)."""
    sh = w.shape
    S, H, dh = sh.seq, sh.heads, sh.head_dim
    Dp, Dm = w.Dp, sh.hidden
    fp = P.fp
    g, Z = fp.g, fp.zeta
    rsq_y, exp_y = P.luts["rsqrt"], P.luts["exp"]
    HS = _p2(H * S)
    dev = w.X.device
    ones_d_col = _ones(Dp, 1, Dm, dev, 0)   # row sums over the valid hidden columns
    ones_d_row = _ones(1, Dp, Dm, dev, 1)   # broadcast to the valid hidden columns
    ones_s_col = _ones(S, 1, S, dev, 0)
    ones_s_row = _ones(1, S, S, dev, 1)

    def div(k):
        return 1 << k

    def matmul(a, b):
        c = _mm(a, b)
        P.matmul(a, b, c)
        return c

    def eprod(a, b):
        c = a.long() * b.long()
        P.eprod(a, b, c)
        return c

    def matadd(a, b, sign=1, dtype=torch.int64):
        c = _add(a, b, sign, dtype)
        P.matadd(a, b, c, sign)
        return c

    def rmsnorm(x):
        """x @g -> (xn @g, u broadcast @g): model.py:640-661's mean square
        (without centring) and the rsqrt lookup, then x * u narrowed."""
        k = _log2(Dp)
        ls = (k + 1) // 2
        var_div = (fp.gamma_fp * Dp) >> (2 * ls)
        xs = P.rescale(x, div(ls))                       # @g-ls
        sq = eprod(xs, xs)                               # @2g-2ls
        ss = matmul(sq, ones_d_col)                      # row sums
        v = P.rescale(ss, var_div).to(torch.int32)       # mean square @g
        u = _lut(rsq_y, v, 0).to(torch.int32)
        P.rsqrt(v, u)
        ub = matmul(u, ones_d_row).to(torch.int32)       # broadcast, padded columns 0
        return P.rescale(eprod(x, ub), Z), ub            # @g

    def project(x, e_x, p, e_out):
        """x W_p (+ (x A_p) B_p) for x @e_x, narrowed to @e_out; returns
        (y, t) with the LoRA hidden t @e_x-1 (A @g-1, B @eW+1)."""
        wide = matmul(x, w.W[p])                         # @e_x+eW
        t = None
        if p in sh.lora:
            t = P.rescale(matmul(x, w.A[p]), Z)
            wide = matadd(wide, matmul(t, w.B[p]))
        return P.rescale(wide, div(e_x + w.eW[p] - e_out)), t

    # ---------------- forward ----------------
    xn, u1 = rmsnorm(w.X)
    q, tq = project(xn, g, "q", g - 1)
    k, tk = project(xn, g, "k", g - 1)
    v, tv = project(xn, g, "v", g - 1)
    qc = P.rescale(eprod(q, w.Cq), Z)                    # q / sqrt(dh) @g-2
    qh, kh, vh = _heads(qc, H, dh), _heads(k, H, dh), _heads(v, H, dh)
    khT = [_t(x) for x in kh]
    zw = [matmul(qh[h], khT[h]) for h in range(H)]       # @2g-3
    lb = fp.exp_base.bit_length() - 1                    # scores @g-lb (|z| < 2^(15-g+lb))
    z = P.rescale(_stack_rows(zw, HS), div(g - 3 + lb))
    del zw
    # softmax: shift by the row max (computed), exp lookup, normalisation
    m = z.max(dim=1, keepdim=True).values.to(torch.int32)
    mb = matmul(m, ones_s_row)
    sv = matadd(mb, z, -1, torch.int32)                  # in [0, 2^16): the table domain
    e = _lut(exp_y, sv, 0).to(torch.int32)               # @g
    P.exp_lookup(sv, e)
    rs = matmul(e, ones_s_col)
    inv = torch.div(fp.gamma_fp * Z + rs // 2, rs, rounding_mode="floor").to(torch.int32)
    invb = matmul(inv, ones_s_row).to(torch.int32)
    pr = P.rescale(eprod(e, invb), Z)                    # @g
    del sv, mb, e, invb
    ph = [pr[h * S:(h + 1) * S].contiguous() for h in range(H)]
    ow = torch.zeros((S, Dp), dtype=torch.int64, device=dev)
    for h in range(H):
        ow[:, h * dh:(h + 1) * dh] = matmul(ph[h], vh[h])  # @2g-1
    o = P.rescale(ow, Z)                                 # @g-1 (o ~ rows of v when p peaks)
    out, to = project(o, g - 1, "o", g)
    x1 = matadd(w.X, out, 1, torch.int16)
    xn2, u2 = rmsnorm(x1)
    gw = matmul(xn2, w.Wg)                               # @2g-1
    act = P.swiglu(gw, "phi")                            # @g-1
    up = P.rescale(matmul(xn2, w.Wu), Z)                 # @g-3
    hh = P.rescale(eprod(act, up), Z)                    # @g-4
    P.rescale(matmul(hh, w.Wd), Z)                       # @g-4

    # ---------------- backward ----------------
    dh_ = P.rescale(matmul(w.dY, _t(w.Wd)), Z)           # @g
    dact = P.swiglu(gw, "phi_prime")                     # @g-1
    du = P.rescale(eprod(dh_, act), div(g - 2))          # @g+1
    dga = P.rescale(eprod(dh_, up), div(g - 3))          # @g
    dg = P.rescale(eprod(dga, dact), Z)                  # @g-1
    a12 = matadd(matmul(dg, _t(w.Wg)), matmul(du, _t(w.Wu)))  # @2g-2
    dxn2 = P.rescale(a12, div(g - 2))                    # @g
    dx1 = matadd(w.dY, P.rescale(eprod(dxn2, u2), Z), 1, torch.int16)

    grads = {}  # LoRA gradients: name -> (tensor, exponent)

    def lora_grads(p, lin, e_lin, t, e_t, dout, e_dout):
        """G = dout B^T, dA = lin^T G, dB = t^T dout, each narrowed by zeta
        (exponents tracked); returns G."""
        e_gp = e_dout + w.eB[p] - g
        gp = P.rescale(matmul(dout, _t(w.B[p])), Z)
        grads["A" + p] = (P.rescale(matmul(_t(lin), gp), Z), e_lin + e_gp - g)
        grads["B" + p] = (P.rescale(matmul(_t(t), dout), Z), e_t + e_dout - g)
        return gp

    dow = matmul(dx1, _t(w.W["o"]))                      # @2g
    if "o" in sh.lora:
        go = lora_grads("o", o, g - 1, to, g - 2, dx1, g)
        dow = matadd(dow, matmul(go, _t(w.A["o"])))
    do = P.rescale(dow, Z)                               # @g
    doh = _heads(do, H, dh)
    dpw, dvw = [], torch.zeros((S, Dp), dtype=torch.int64, device=dev)
    for h in range(H):
        dpw.append(matmul(doh[h], _t(vh[h])))           # @2g-1
        dvw[:, h * dh:(h + 1) * dh] = matmul(_t(ph[h]), doh[h])  # @2g
    dp = P.rescale(_stack_rows(dpw, HS), div(g - 1))     # @g
    del dpw
    dv = P.rescale(dvw, Z)                               # @g
    # softmax backward (model.py:785-791): dz = p * (dp - rowsum(dp * p))
    w1 = P.rescale(eprod(dp, pr), Z)
    rsb = matmul(matmul(w1, ones_s_col), ones_s_row)
    dd = matadd(dp, rsb, -1, torch.int16)
    dz = P.rescale(eprod(pr, dd), Z)                     # @g
    del w1, rsb, dd
    dqcw = torch.zeros((S, Dp), dtype=torch.int64, device=dev)
    dkw = torch.zeros((S, Dp), dtype=torch.int64, device=dev)
    for h in range(H):
        dzh = dz[h * S:(h + 1) * S].contiguous()
        dqcw[:, h * dh:(h + 1) * dh] = matmul(dzh, kh[h])    # @2g-1
        dkw[:, h * dh:(h + 1) * dh] = matmul(_t(dzh), qh[h])  # @2g-2
    dqc = P.rescale(dqcw, div(g - 1))                    # @g
    dq = P.rescale(eprod(dqc, w.Cq), div(g - 1))         # @g
    dk = P.rescale(dkw, div(g - 2))                      # @g
    gq = {"q": dq, "k": dk, "v": dv}
    hidden = {"q": tq, "k": tk, "v": tv}
    dxw = None
    for p in "qkv":
        c = matmul(gq[p], _t(w.W[p]))                    # @2g-1
        dxw = c if dxw is None else matadd(dxw, c)
        if p in sh.lora:
            gp = lora_grads(p, xn, g, hidden[p], g - 1, gq[p], g)
            dxw = matadd(dxw, matmul(gp, _t(w.A[p])))
    dxn = P.rescale(dxw, div(g - 1))                     # @g
    P.rescale(eprod(dxn, u1), Z)

    # ---------------- LoRA update (model.py:823-836) ----------------
    # step = grad / (eta_div * 2^(e_grad - e_w)) lands on the weight's exponent
    for p in sh.lora:
        for name, W_, e_w in (("A", w.A[p], w.eA), ("B", w.B[p], w.eB[p])):
            gt, e_g = grads[name + p]
            d = fp.eta_div << (e_g - e_w) if e_g >= e_w else fp.eta_div >> (e_w - e_g)
            matadd(W_, P.rescale(gt, d), -1, torch.int16)
    return P


def summary(P):
    """Census of one proven block: per gadget kind (count, rounds, field
    elements, seconds) and totals."""
    kinds = {k: {"count": v[0], "rounds": v[1], "field_elems": v[2], "seconds": v[3]}
             for k, v in sorted(P.stats.items())}
    tot = {"count": sum(v[0] for v in P.stats.values()),
           "rounds": sum(v[1] for v in P.stats.values()),
           "field_elems": sum(v[2] for v in P.stats.values()),
           "seconds": sum(v[3] for v in P.stats.values())}
    return {"gadgets": kinds, "total": tot, "clipped_quotients": 0}
