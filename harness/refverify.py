"""Verifier in the loop: the REFERENCE's own verifiers judge this backend's
proofs.

The reference package comes from baseline/_ref (a pip --target install of
/root/reference/pkg; git-ignored, it travels to the GPU box with the repo).
`BlockVerifier` is a BlockProver.on_proof hook: right after each gadget is
proven it runs the matching reference verifier

    verify_matmul      gadgets.py:268-309     verify_matadd     gadgets.py:339-367
    verify_elementprod gadgets.py:413-444     verify_rescale    gadgets.py:625-652
    verify_swiglu      gadgets.py:783-811     verify_rsqrt      gadgets.py:850-858
    _verify_pair_lookup gadgets.py:691-698    (verify_lookup    lookup.py:254-318)

on the reference's own Transcript class (hashlib SHAKE-256), which therefore
stays in lockstep with the prover's native transcript; the end states must
be equal.

Commitments are out of scope (BASELINE north star), so both sides use the
deterministic stub (paper_2508_21393_b200/commit_stub.py).  A stub binds
nothing, so `OpeningChecker` stands in for the commitment check: every stub
commitment carries a handle on what it commits to (commit_stub.CHECK), and
every opened value the verifier consumes is recomputed independently of the
prover --

  * tensor operands and table columns: lifted and folded to the point
    (zkl_lift + zkl_fold chain, not the sumcheck engine that produced the
    prover's finals);
  * logUp helper columns 1/(beta + s): a fresh batch inversion of the
    secret itself (the prover gathers them through the table index);
  * multiplicities: torch sort / searchsorted / bincount over canonical
    field elements (the prover bins with its own atomics kernels);
  * combined pair commitments: the same linear combination of the parts.

A mismatch makes verify_batch return False, so the reference verifier
rejects.  This module is a test / measurement harness: nothing in the
package imports it.
"""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2508_21393_b200 import _native as N  # noqa: E402
from paper_2508_21393_b200 import commit_stub as CS  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402
from paper_2508_21393_b200.field import batch_inverse_device  # noqa: E402
from paper_2508_21393_b200.gadgets import DeviceMatrix  # noqa: E402
from paper_2508_21393_b200.mle import mle_evaluate_device  # noqa: E402


def reference_available():
    return os.path.isdir(os.path.join(REF, "zklora"))


def load_reference():
    """The reference modules (gadgets, lookup, tables, transcript)."""
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import zklora.gadgets as G
    import zklora.lookup as L
    import zklora.tables as TB
    import zklora.transcript as T

    return G, L, TB, T


class StubGroupKey:
    """The verifier-side key: only .group is read (None for the stub)."""

    group = None


# ---------------------------------------------------------------------------
class OpeningChecker:
    """verify_batch for stub commitments: the transcript traffic of
    commit_stub.open_batch, plus an independent evaluation of every opened
    value from the commitment's handle."""

    def __init__(self, spec):
        self.spec = spec
        self.p = spec.modulus
        self.checked = 0
        self.unchecked = 0
        self.failures = []

    # --- field buffers of the things commitments stand for -----------------
    def _field(self, obj):
        """(device field buffer, n) of a DeviceMatrix / int column / device
        vector / list of residues."""
        spec = self.spec
        if isinstance(obj, DeviceMatrix):
            if obj.mtype == N.MT_FIELD:
                return obj.t, obj.rows * obj.cols
            return D.lift(obj.t.reshape(-1), spec), obj.rows * obj.cols
        if torch.is_tensor(obj):
            if obj.dtype in (torch.int16, torch.int32, torch.int64) and obj.dim() == 1:
                return D.lift(obj, spec), obj.numel()
            raise TypeError("unsupported tensor handle %s %s" % (obj.dtype, tuple(obj.shape)))
        if isinstance(obj, D.LiftedColumn):
            return D.lift(obj.col, spec), obj.n
        if isinstance(obj, D.PairColumn):
            return D.pair_combine(obj.x, obj.y, obj.alpha, spec).buf, obj.n
        if isinstance(obj, D.DeviceVector):
            return obj.buf, obj.n
        vals = list(obj)
        return D.upload(vals, spec), len(vals)

    def _canonical(self, buf, n):
        """Canonical little-endian words (n, W) int64 (zkl_from_mont)."""
        spec = self.spec
        out = D.empty(spec, n)
        N.check(N.lib().zkl_from_mont(spec.fid, D.ptr(out), D.ptr(buf), n, D.stream()))
        return out[:n].view(n, spec.words)

    def _multiplicities(self, entries, table_entries):
        """compute_multiplicities (lookup.py:91-99) by sorting: each secret
        entry counts to the LAST table index holding its value."""
        sb, d = self._field(entries)
        tb, n = self._field(table_entries)
        S, T = self._canonical(sb, d), self._canonical(tb, n)
        mix = torch.tensor([0x9E3779B97F4A7C15 - (1 << 64), 0x632BE59BD9B4E019,
                            0x3C6EF372FE94F82B, 0x1B873593CC9E2D51][: S.shape[1]],
                           dtype=torch.int64, device=S.device)

        def key(X):
            return (X * mix).sum(1)  # wrapping int64 arithmetic

        tk = key(T)
        order = torch.sort(tk, stable=True)
        sk = key(S)
        pos = torch.searchsorted(order.values, sk, right=True) - 1
        pos = pos.clamp_(min=0)
        idx = order.indices[pos]
        if not bool((T[idx] == S).all()):
            return None  # an entry outside the table: the claim is false
        return torch.bincount(idx, minlength=n)

    # --- MLE of a handle at a point -----------------------------------------
    def mle(self, handle, point):
        spec, p = self.spec, self.p
        if isinstance(handle, tuple) and handle and handle[0] == "lin":
            return sum(c * self.mle(h, point) for h, c in handle[1]) % p
        if isinstance(handle, tuple) and handle and handle[0] == "inv":
            _, entries, beta = handle
            buf, n = self._field(entries)
            inv, zero = batch_inverse_device(buf, n, spec, add=beta)
            if zero is not None:
                return None
            return mle_evaluate_device(inv, len(point), list(point), spec)
        if isinstance(handle, tuple) and handle and handle[0] == "mult":
            _, entries, table_entries, _prover_m = handle
            m = self._multiplicities(entries, table_entries)
            if m is None:
                return None
            return mle_evaluate_device(D.lift(m, spec), len(point), list(point), spec)
        buf, n = self._field(handle)
        if n != 1 << len(point):
            return None
        return mle_evaluate_device(buf, len(point), list(point), spec)

    def verify_batch(self, key, commitments, point, values, proof, tr):
        for r in point:
            tr.append(b"open/point", r)
        for v in values:
            tr.append(b"open/value", v)
        if len(commitments) != len(values):
            return False
        ok = True
        for c, v in zip(commitments, values):
            h = getattr(c, "handle", None)
            if h is None:
                self.unchecked += 1
                continue
            got = self.mle(h, point)
            self.checked += 1
            if got is None or got != v % self.p:
                ok = False
                self.failures.append((type(h).__name__ if not isinstance(h, tuple) else h[0],
                                      len(point)))
        return ok


# ---------------------------------------------------------------------------
def reference_tables(tables, spec, TB, L):
    """The reference's TableSet (tables.py:156-168) over a block's device
    tables: Python-int entries, the same stub commitments (same bytes), each
    with a handle on its device column for the opening checks."""
    from dataclasses import replace

    p = spec.modulus

    def ints(col):
        return tuple(int(v) % p for v in col.tolist())

    def col(entries, com, name):
        return L.LookupTable(ints(entries), replace(com, handle=entries), name)

    def single(t):
        return col(t.int_column, t.commitment, t.name)

    def pair(pt):
        return TB.PairTable(col(pt.x.entries, pt.x.commitment, pt.x.name),
                            col(pt.y.entries, pt.y.commitment, pt.y.name), pt.name)

    return TB.TableSet(tables.params, tables.eps, p, b"",
                       tuple(pair(e) for e in tables.exp_segments), pair(tables.silu),
                       pair(tables.silu_deriv), pair(tables.rsqrt), single(tables.quant_range),
                       single(tables.residue_range))


class BlockVerifier:
    """BlockProver.on_proof hook running the reference verifiers in lockstep
    (module docstring).  Requires commit_stub.CHECK = True while proving."""

    def __init__(self, tables, spec, domain, seed):
        G, L, TB, T = load_reference()
        self.G = G
        self.spec = spec
        self.tr = T.Transcript(domain, spec.modulus, seed)
        self.checker = OpeningChecker(spec)
        # the stub commitment path on the reference side (as in
        # tests/golden/make_golden.py), with the checking verify_batch
        for mod in (G, L):
            mod.verify_batch = self.checker.verify_batch
        G.combine_commitments = CS.combine_commitments
        TB.combine_commitments = CS.combine_commitments
        self.ts = reference_tables(tables, spec, TB, L)
        self.key = StubGroupKey()
        self.results = []

    def __call__(self, kind, refs, proof, extra=None):
        G, ts, key, tr = self.G, self.ts, self.key, self.tr
        if kind == "matmul":
            ok = G.verify_matmul(*refs, proof, key, tr)
        elif kind == "matadd":
            ok = G.verify_matadd(*refs, proof, key, tr)
        elif kind == "elementprod":
            ok = G.verify_elementprod(*refs, proof, key, tr)
        elif kind == "rescale":
            ok = G.verify_rescale(*refs, proof, ts, key, tr)
        elif kind == "swiglu":
            ok = G.verify_swiglu(refs[0], refs[1], proof, ts, key, tr)
        elif kind == "rsqrt":
            ok = G.verify_rsqrt(refs[0], refs[1], proof, ts, key, tr)
        elif kind == "softmax_exp":
            ok = G._verify_pair_lookup(b"softmax/exp0", refs[0], refs[1], ts.exp_segments[0],
                                       proof, key, tr)
        else:
            raise ValueError("no reference verifier for %r" % kind)
        self.results.append((kind, bool(ok)))

    def summary(self):
        rejected = [i for i, (_, ok) in enumerate(self.results) if not ok]
        return {"gadgets_verified": len(self.results), "rejected": len(rejected),
                "first_rejected": (self.results[rejected[0]][0], rejected[0]) if rejected
                else None,
                "openings_checked": self.checker.checked,
                "openings_unchecked": self.checker.unchecked,
                "opening_mismatches": len(self.checker.failures),
                "verifier_accept": bool(self.results) and not rejected}


def prove_and_verify_block(w, tables, spec, domain, seed):
    """Prove a block with the reference verifiers in the loop.  Returns
    (BlockProver, BlockVerifier summary dict with 'transcripts_equal')."""
    from paper_2508_21393_b200 import block as BK
    from paper_2508_21393_b200.transcript import Transcript

    prev = CS.CHECK
    CS.CHECK = True
    try:
        V = BlockVerifier(tables, spec, domain, seed)
        tr = Transcript(domain, spec.modulus, seed)
        P = BK.prove_block(w, BK.BlockProver(tr, tables, timing=False, on_proof=V))
    finally:
        CS.CHECK = prev
    s = V.summary()
    s["transcripts_equal"] = bytes(tr.state) == bytes(V.tr.state)
    s["verifier_accept"] = s["verifier_accept"] and s["transcripts_equal"]
    return P, s
