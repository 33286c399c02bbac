"""LoRA transformer-block proof schedule (BASELINE configs 4/5, "LoRA-block
proof seconds"), composed from this backend's gadget provers.

The reference cannot express these blocks (SURVEY.md sec. 7 hard part 6:
pow-2 dims only, single head, LayerNorm, LoRA on W_V only), so the schedule is
a new composition of the reference's gadget API, every instance proven by the
drop-ins here on one sequential Fiat-Shamir transcript:

  prove_matmul       gadgets.py:230-265   every fwd / bwd / LoRA-gradient matmul
  prove_elementprod  gadgets.py:383-410   RMSNorm scaling, softmax normalisation,
                                          SwiGLU gate products and their gradients
  prove_rescale      gadgets.py:600-622   every wide -> int16 narrowing
  prove_swiglu       gadgets.py:761-782   SiLU / SiLU' of the gate (phi, phi_prime)
  prove_rsqrt        gadgets.py:842-847   RMSNorm 1/sqrt(mean square)
  _prove_pair_lookup gadgets.py:679-688   softmax: row-max-shifted exp, one 2^16
                                          segment (BASELINE cfg4)

Witnesses are seeded synthetic fixed-point tensors (int16 at gamma = zeta =
2^12, act_bound 8): X ~ N(0,1), weights ~ N(0,0.02) (W_q carries the
1/sqrt(d_head) score scale), dY ~ N(0,1e-2).  They are
chained through an exact fixed-point forward and backward pass on the GPU
(int64 products via float64 GEMMs, |partial sums| < 2^53), so every gadget's
claim is honest for its operands.  Dimensions that are not powers of two are
zero-padded (quantize.py:176-183); the padded attention rows use the valid
exp pair (0, gamma).  Not proven here (they are openings or public
arithmetic in the reference, or outside this path): matadd (residual adds,
LoRA sums), the softmax row-sum reciprocal and the RMSNorm mean-square
reduction (inputs to the proven elementprod / rsqrt), the AdamW/SGD update.
Commitments use the deterministic stub (commit_stub.py).
"""

import time
from collections import defaultdict
from dataclasses import dataclass

import numpy as np
import torch

from . import tables as TBL
from .commit_stub import StubCommitment, StubKey
from .gadgets import DeviceMatrix, ProverTensor, TensorRef, prove_elementprod, prove_matmul
from .gadgets import prove_pair_lookup
from .nonlinear import (TableSet, device_pair_table, device_range_table,
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
    2^12, act_bound 8, one 2^16 exp segment, RMSNorm eps 1e-5."""

    gamma_fp: int = 1 << 12
    zeta: int = 1 << 12
    act_bound: int = 8
    exp_n: int = 1 << 16
    eps: float = 1e-5

    @property
    def qmin(self):
        return -self.act_bound * self.gamma_fp

    @property
    def qmax(self):
        return self.act_bound * self.gamma_fp - 1


FP = FixedPoint()


def _p2(n):
    return 1 << (n - 1).bit_length()


def _log2(n):
    return (n - 1).bit_length()


def block_tables(spec, fp=FP):
    """The TableSet of the block (tables.py:217-238 fields) on the device."""
    g, a = fp.gamma_fp, fp.act_bound

    def com(n):
        return StubCommitment(_log2(n))

    lo, n = TBL.quant_range(g, a)
    quant = device_range_table(lo, n, spec, com(n), "quant_range")
    lo, n = TBL.residue_range(fp.zeta)
    resid = device_range_table(lo, n, spec, com(n), "residue_range")

    def pair(cols, name):
        c = com(len(cols[0]))
        return device_pair_table(*cols, c, c, name)

    return TableSet(fp, fp.eps, spec.modulus, b"", (
        pair(TBL.exp_segment_entries(g, (fp.exp_n,), 0), "exp0"),),
        pair(TBL.silu_entries(g, a), "silu"), pair(TBL.silu_deriv_entries(g, a), "silu_deriv"),
        pair(TBL.rsqrt_entries(g, a, fp.eps), "rsqrt"), quant, resid)


def block_luts(tables):
    """Witness-side table outputs (int32 columns) keyed by name."""
    return {"silu": tables.silu.y.entries, "silu_deriv": tables.silu_deriv.y.entries,
            "rsqrt": tables.rsqrt.y.entries, "exp": tables.exp_segments[0].y.entries}


# ---------------------------------------------------------------------------
# fixed-point witness arithmetic (device, untimed)
def _q16(rng, shape, std, rows, cols, gamma, device):
    """round_half_away(N(0,std) * gamma) clipped to int16, zero-padded to
    (rows, cols)."""
    a = rng.standard_normal(shape) * std * gamma
    a = np.clip(np.sign(a) * np.floor(np.abs(a) + 0.5), -32768, 32767).astype(np.int16)
    t = torch.zeros((rows, cols), dtype=torch.int16)
    t[: shape[0], : shape[1]] = torch.from_numpy(a)
    return t.to(device)


def _mm(a, b):
    """Exact int64 a @ b of int16 matrices (float64 GEMM; |sums| < 2^53)."""
    assert a.shape[1] * (1 << 30) < (1 << 53)
    return torch.matmul(a.double(), b.double()).round_().long()


def _divmod(wide, fp):
    """centered_divmod (quantize.py:101-104) with the quotient clipped to the
    quant_range domain; returns (q int16, r int16, clipped count).  On the GPU
    one fused pass (nonlinear.rescale_witness_device); the torch form below is
    the CPU path the golden generator drives the reference with."""
    if wide.is_cuda:
        return rescale_witness_device(wide, fp.zeta, fp, clip=True)
    d = fp.zeta
    q = torch.div(wide + d // 2, d, rounding_mode="floor")
    r = (wide - d * q).to(torch.int16)
    clipped = int(((q < fp.qmin) | (q > fp.qmax)).sum())
    return q.clamp_(fp.qmin, fp.qmax).to(torch.int16), r, clipped


def _lut(table_y, x, x0):
    return table_y[(x.long() - x0)]


class BlockProver:
    """One sequential transcript over the whole block; records per-gadget
    counts, rounds, field elements and seconds."""

    def __init__(self, tr, tables, key=None, timing=True):
        self.tr, self.tables = tr, tables
        self.timing = timing  # per-gadget synchronised spans (off: the host runs ahead)
        self.fp = tables.params
        self.luts = block_luts(tables)
        self.key = key or StubKey()
        self.stats = defaultdict(lambda: [0, 0, 0, 0.0])  # count, rounds, elems, seconds
        self.clipped = 0
        self.log = []  # [kind, rounds of each sumcheck] per gadget, in proof order
        self.seconds = []  # per gadget, same order as log

    class _Rng:
        def vector(self, n):
            return [0] * n

    def pt(self, t):
        rv, cv = _log2(t.shape[0]), _log2(t.shape[1])
        ref = TensorRef("committed", rv, cv, commitment=StubCommitment(rv + cv))
        return ProverTensor(None, ref, (), device=DeviceMatrix.from_int_tensor(t))

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

    def matmul(self, a, b, c):
        pr = self._run("matmul", prove_matmul, self.pt(a), self.pt(b), self.pt(c), self.key,
                       self.tr, self._Rng())
        n = sum(pr.dims)
        self._count("matmul", n, 4 << n)
        self.log.append(["matmul", len(pr.sumcheck.rounds)])
        return pr

    def eprod(self, a, b, c):
        pr = self._run("elementprod", prove_elementprod, self.pt(a), self.pt(b), self.pt(c),
                       self.key, self.tr, self._Rng())
        n = sum(pr.shape)
        self._count("elementprod", n, 3 << n)
        self.log.append(["elementprod", len(pr.sumcheck.rounds)])
        return pr

    def _lookups(self, kind, lps):
        self.log.append([kind] + [len(lp.sumcheck.rounds) for lp in lps])
        for lp in lps:
            n = len(lp.sumcheck.rounds)
            self._count(kind, n, 7 << n)

    def rescale(self, wide):
        q, r, clipped = _divmod(wide, self.fp)
        self.clipped += clipped
        self.rescale_w(wide, q, r)
        return q

    def rescale_w(self, wide, q, r):
        pr = self._run("rescale", prove_rescale, self.pt(wide), self.pt(q), self.pt(r),
                       self.fp.zeta, self.tables, self.key, self.tr, self._Rng())
        self._lookups("rescale", (pr.quant_lookup, pr.resid_lookup))

    def swiglu(self, wide, mode):
        q, r, clipped = _divmod(wide, self.fp)
        self.clipped += clipped
        table = self.luts["silu" if mode == "phi" else "silu_deriv"]
        out = _lut(table, q, self.fp.qmin).to(torch.int16)
        self.swiglu_w(wide, out, q, r, mode)
        return out

    def swiglu_w(self, wide, out, q, r, mode):
        pr = self._run("swiglu", prove_swiglu, self.pt(wide), self.pt(out), self.pt(q),
                       self.pt(r), mode, self.tables, self.key, self.tr, self._Rng())
        self._lookups("swiglu", (pr.activation_lookup, pr.resid_lookup))

    def rsqrt(self, v, u):
        pr = self._run("rsqrt", prove_rsqrt, self.pt(v), self.pt(u), self.tables, self.key,
                       self.tr, self._Rng())
        self._lookups("rsqrt", (pr.lookup,))

    def exp_lookup(self, v, e):
        pr = self._run("softmax_exp", prove_pair_lookup, b"softmax/exp0", self.pt(v),
                       self.pt(e), self.tables.exp_segments[0], self.key, self.tr, self._Rng())
        self._lookups("softmax_exp", (pr,))


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
        self.clipped = 0

    def matmul(self, a, b, c):
        self.calls.append(("matmul", a, b, c))

    def eprod(self, a, b, c):
        self.calls.append(("eprod", a, b, c))

    def rescale(self, wide):
        q, r, clipped = _divmod(wide, self.fp)
        self.clipped += clipped
        self.calls.append(("rescale_w", wide, q, r))
        return q

    def swiglu(self, wide, mode):
        q, r, clipped = _divmod(wide, self.fp)
        self.clipped += clipped
        table = self.luts["silu" if mode == "phi" else "silu_deriv"]
        out = _lut(table, q, self.fp.qmin).to(torch.int16)
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
        P.clipped = self.clipped
        return P


# ---------------------------------------------------------------------------
class BlockWitness:
    """Seeded weights and input of one block, padded to powers of two."""

    def __init__(self, shape, seed=0, fp=FP, device="cuda"):
        self.shape = shape
        g = np.random.Generator(np.random.PCG64(seed))
        S, Dm, F, R = shape.seq, shape.hidden, shape.ffn, shape.rank
        Dp, Fp = _p2(Dm), _p2(F)
        self.Dp, self.Fp = Dp, Fp

        def q(sh, std, rows, cols):
            return _q16(g, sh, std, rows, cols, fp.gamma_fp, device)

        self.X = q((S, Dm), 1.0, S, Dp)
        # the attention score scale 1/sqrt(d_head) is folded into W_q
        self.W = {p: q((Dm, Dm), 0.02 / (shape.head_dim ** 0.5 if p == "q" else 1.0), Dp, Dp)
                  for p in "qkvo"}
        self.Wg = q((Dm, F), 0.02, Dp, Fp)
        self.Wu = q((Dm, F), 0.02, Dp, Fp)
        self.Wd = q((F, Dm), 0.02, Fp, Dp)
        self.A = {p: q((Dm, R), 0.02, Dp, R) for p in shape.lora}
        self.B = {p: q((R, Dm), 0.02, R, Dp) for p in shape.lora}
        self.dY = q((S, Dm), 1e-2, S, Dp)


def _t(x):
    return x.t().contiguous()


def _heads(x, H, dh):
    return [x[:, h * dh:(h + 1) * dh].contiguous() for h in range(H)]


def _stack_rows(mats, rows):
    """Stack (S x C) matrices vertically and zero-pad to `rows` rows."""
    out = torch.zeros((rows, mats[0].shape[1]), dtype=mats[0].dtype, device=mats[0].device)
    torch.cat(mats, out=out[: sum(m.shape[0] for m in mats)])
    return out


def _clip16(x):
    return x.clamp(-32768, 32767).to(torch.int16)


def prove_block(w, P):
    """Prove one LoRA fine-tuning step of one transformer block (forward,
    backward, LoRA gradients) through the gadget prover P (BlockProver, or a
    stand-in with the same methods that drives the reference's gadgets for
    parity goldens).  Returns P."""
    sh = w.shape
    S, H, dh = sh.seq, sh.heads, sh.head_dim
    Dp = w.Dp
    fp = P.fp
    G, Z = fp.gamma_fp, fp.zeta
    rsq_y, exp_y = P.luts["rsqrt"], P.luts["exp"]
    HS = _p2(H * S)
    Dm = sh.hidden
    dev = w.X.device

    def rmsnorm(x):
        """u = rsqrt(mean(x^2)) per row (proven lookup), x * u (elementprod),
        narrowed.  Returns (xn, u broadcast)."""
        ms = (x.double() ** 2).sum(1, keepdim=True) / Dm / G  # mean square at gamma
        v = torch.clamp(torch.floor(ms + 0.5), 0, fp.qmax).to(torch.int32)
        u = _lut(rsq_y, v, 0).to(torch.int32)
        P.rsqrt(v, u)
        ub = u.expand(-1, Dp).contiguous()
        if Dp != Dm:
            ub[:, Dm:] = 0
        wide = x.long() * ub.long()
        P.eprod(x, ub, wide)
        return P.rescale(wide), ub

    def project(x, p, lora_in):
        """x W_p (+ (x A_p) B_p); returns (y, t) with t the LoRA hidden."""
        wide = _mm(x, w.W[p])
        P.matmul(x, w.W[p], wide)
        t = None
        if p in sh.lora:
            tw = _mm(lora_in, w.A[p])
            P.matmul(lora_in, w.A[p], tw)
            t = P.rescale(tw)
            lw = _mm(t, w.B[p])
            P.matmul(t, w.B[p], lw)
            wide = wide + lw  # matadd (opening only in the reference)
        return P.rescale(wide), t

    # ---------------- forward ----------------
    xn, u1 = rmsnorm(w.X)
    q, tq = project(xn, "q", xn)
    k, tk = project(xn, "k", xn)
    v, tv = project(xn, "v", xn)
    qh, kh, vh = _heads(q, H, dh), _heads(k, H, dh), _heads(v, H, dh)
    khT = [_t(x) for x in kh]
    zw = []
    for h in range(H):
        c = _mm(qh[h], khT[h])
        P.matmul(qh[h], khT[h], c)
        zw.append(c)
    z = P.rescale(_stack_rows(zw, HS))
    del zw
    # softmax: row-max-shifted exp lookup, normalisation elementprod
    m = z.max(dim=1, keepdim=True).values.long()
    sv = torch.clamp(m - z.long(), 0, fp.exp_n - 1).to(torch.int32)
    sv[H * S:] = 0  # padded rows: the valid pair (0, gamma)
    e = _lut(exp_y, sv, 0).to(torch.int32)
    P.exp_lookup(sv, e)
    rs = e.long().sum(1, keepdim=True)
    inv = torch.div(G * Z + rs // 2, rs, rounding_mode="floor").to(torch.int32)
    invb = inv.expand(-1, S).contiguous()
    pw = e.long() * invb.long()
    P.eprod(e, invb, pw)
    pr = P.rescale(pw)
    del pw, invb, e, sv
    ph = [pr[h * S:(h + 1) * S].contiguous() for h in range(H)]
    ow = torch.zeros((S, Dp), dtype=torch.int64, device=dev)
    for h in range(H):
        c = _mm(ph[h], vh[h])
        P.matmul(ph[h], vh[h], c)
        ow[:, h * dh:(h + 1) * dh] = c
    o = P.rescale(ow)
    out, to = project(o, "o", o)
    x1 = _clip16(w.X.int() + out.int())
    xn2, u2 = rmsnorm(x1)
    gw = _mm(xn2, w.Wg)
    P.matmul(xn2, w.Wg, gw)
    uw = _mm(xn2, w.Wu)
    P.matmul(xn2, w.Wu, uw)
    act = P.swiglu(gw, "phi")
    up = P.rescale(uw)
    hw = act.long() * up.long()
    P.eprod(act, up, hw)
    hh = P.rescale(hw)
    dw = _mm(hh, w.Wd)
    P.matmul(hh, w.Wd, dw)
    P.rescale(dw)

    # ---------------- backward ----------------
    WdT = _t(w.Wd)
    dhw = _mm(w.dY, WdT)
    P.matmul(w.dY, WdT, dhw)
    dh_ = P.rescale(dhw)
    dact = P.swiglu(gw, "phi_prime")
    duw = dh_.long() * act.long()
    P.eprod(dh_, act, duw)
    du = P.rescale(duw)
    dgaw = dh_.long() * up.long()
    P.eprod(dh_, up, dgaw)
    dga = P.rescale(dgaw)
    dgw = dga.long() * dact.long()
    P.eprod(dga, dact, dgw)
    dg = P.rescale(dgw)
    WgT, WuT = _t(w.Wg), _t(w.Wu)
    a1 = _mm(dg, WgT)
    P.matmul(dg, WgT, a1)
    a2 = _mm(du, WuT)
    P.matmul(du, WuT, a2)
    dxn2 = P.rescale(a1 + a2)
    d1w = dxn2.long() * u2.long()
    P.eprod(dxn2, u2, d1w)
    dx1 = _clip16(w.dY.int() + P.rescale(d1w).int())

    def lora_grads(p, lin, t, dout):
        """G = dout B^T, dA = lin^T G, dB = t^T dout; returns G."""
        BT = _t(w.B[p])
        gw_ = _mm(dout, BT)
        P.matmul(dout, BT, gw_)
        gp = P.rescale(gw_)
        linT = _t(lin)
        da = _mm(linT, gp)
        P.matmul(linT, gp, da)
        P.rescale(da)
        tT = _t(t)
        db = _mm(tT, dout)
        P.matmul(tT, dout, db)
        P.rescale(db)
        return gp

    WoT = _t(w.W["o"])
    dow = _mm(dx1, WoT)
    P.matmul(dx1, WoT, dow)
    if "o" in sh.lora:
        go = lora_grads("o", o, to, dx1)
        AoT = _t(w.A["o"])
        c = _mm(go, AoT)
        P.matmul(go, AoT, c)
        dow = dow + c
    do = P.rescale(dow)
    doh = _heads(do, H, dh)
    dpw, dvw = [], torch.zeros((S, Dp), dtype=torch.int64, device=dev)
    for h in range(H):
        vT = _t(vh[h])
        c = _mm(doh[h], vT)
        P.matmul(doh[h], vT, c)
        dpw.append(c)
        pT = _t(ph[h])
        c = _mm(pT, doh[h])
        P.matmul(pT, doh[h], c)
        dvw[:, h * dh:(h + 1) * dh] = c
    dp = P.rescale(_stack_rows(dpw, HS))
    del dpw
    dv = P.rescale(dvw)
    # softmax backward: dZ = P * (dP - rowdot(P, dP))
    rowdot = torch.div((pr.long() * dp.long()).sum(1, keepdim=True) + G // 2, G,
                       rounding_mode="floor")
    dzin = _clip16(dp.long() - rowdot)
    dzw = pr.long() * dzin.long()
    P.eprod(pr, dzin, dzw)
    dz = P.rescale(dzw)
    del dzw, dzin
    dqw = torch.zeros((S, Dp), dtype=torch.int64, device=dev)
    dkw = torch.zeros((S, Dp), dtype=torch.int64, device=dev)
    for h in range(H):
        dzh = dz[h * S:(h + 1) * S].contiguous()
        c = _mm(dzh, kh[h])
        P.matmul(dzh, kh[h], c)
        dqw[:, h * dh:(h + 1) * dh] = c
        dzT = _t(dzh)
        c = _mm(dzT, qh[h])
        P.matmul(dzT, qh[h], c)
        dkw[:, h * dh:(h + 1) * dh] = c
    dq, dk = P.rescale(dqw), P.rescale(dkw)
    grads = {"q": dq, "k": dk, "v": dv}
    hidden = {"q": tq, "k": tk, "v": tv}
    dxw = torch.zeros((S, Dp), dtype=torch.int64, device=dev)
    for p in "qkv":
        WT = _t(w.W[p])
        c = _mm(grads[p], WT)
        P.matmul(grads[p], WT, c)
        dxw += c
        if p in sh.lora:
            gp = lora_grads(p, xn, hidden[p], grads[p])
            AT = _t(w.A[p])
            c = _mm(gp, AT)
            P.matmul(gp, AT, c)
            dxw += c
    dxn = P.rescale(dxw)
    d0w = dxn.long() * u1.long()
    P.eprod(dxn, u1, d0w)
    P.rescale(d0w)
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
    return {"gadgets": kinds, "total": tot, "clipped_quotients": P.clipped}
