"""Generate golden vectors by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.json.  The reference is imported from
/root/reference (read-only) and never copied; only its outputs on seeded
inputs are committed.  Commitments are replaced on the reference side by
the deterministic stub documented in oracle/stubcommit.py (monkeypatching
zklora.lookup.commit/open_batch and zklora.gadgets.commit/open_batch), so
the transcript bytes are reproducible by a backend that does not implement
Pedersen commitments (out of scope).
"""

import base64
import json
import os
import random
import sys
import time
import zlib
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import inputs  # noqa: E402
import zklora.gadgets as G  # noqa: E402
import zklora.lookup as L  # noqa: E402
from zklora import field as F  # noqa: E402
from zklora import mle as M  # noqa: E402
from zklora.quantize import QuantParams  # noqa: E402
from zklora.sumcheck import SumcheckClaim, Term, direct_sum, prove_sumcheck  # noqa: E402
from zklora import tables as TB  # noqa: E402
from zklora.transcript import Transcript  # noqa: E402

STUB_TAG = b"zkl-stub/v1"


class StubCom:
    def __init__(self, num_vars):
        self.num_vars = num_vars

    def serialize(self, group):
        return STUB_TAG + bytes([self.num_vars])


def stub_commit(key, table, blinding=None):
    return StubCom((len(table) - 1).bit_length())


def stub_open(key, tables, blindings, point, tr, rng):
    p = tr.modulus
    vals = [M.mle_evaluate(list(t), list(point), p) for t in tables]
    for r in point:
        tr.append(b"open/point", r)
    for y in vals:
        tr.append(b"open/value", y)
    return vals, None


def stub_combine(group, commitments, coefficients):
    return StubCom(commitments[0].num_vars)


L.commit = stub_commit
L.open_batch = stub_open
G.commit = stub_commit
G.open_batch = stub_open
G.combine_commitments = stub_combine
TB.combine_commitments = stub_combine
KEY = SimpleNamespace(group=None)
RNG = SimpleNamespace(vector=lambda n: [0] * n, next=lambda: 0)

FIELDS = {"big": F.MODULUS, "test": F.TEST_MODULUS}


def hx(b):
    return b.hex()


def dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


# ---------------------------------------------------------------------------
def gen_transcript():
    cases = []
    rnd = random.Random(1234)
    for fname, p in FIELDS.items():
        for k in range(6):
            domain = b"zkl/golden/%d" % k
            seed = bytes(rnd.randrange(256) for _ in range(rnd.randrange(0, 40)))
            tr = Transcript(domain, p, seed)
            ops, outs = [], []
            for _ in range(12):
                kind = rnd.randrange(4)
                label = b"lbl/" + bytes([97 + rnd.randrange(26)]) * rnd.randrange(1, 30)
                if kind == 0:
                    data = bytes(rnd.randrange(256) for _ in range(rnd.randrange(0, 200)))
                    tr.append(label, data)
                    ops.append(["bytes", hx(label), hx(data)])
                elif kind == 1:
                    v = rnd.randrange(0, p) if rnd.random() < 0.8 else rnd.randrange(0, 300)
                    tr.append(label, v)
                    ops.append(["int", hx(label), v])
                elif kind == 2:
                    c = tr.challenge(label)
                    ops.append(["challenge", hx(label)])
                    outs.append(c)
                else:
                    cnt = rnd.randrange(0, 5)
                    cs = tr.challenge_vector(label, cnt)
                    ops.append(["vector", hx(label), cnt])
                    outs.extend(cs)
            cases.append(
                dict(field=fname, domain=hx(domain), seed=hx(seed), ops=ops,
                     challenges=outs, state=hx(tr.state))
            )
    dump("transcript.json", cases)


# ---------------------------------------------------------------------------
def _rand_terms(rnd, k, degree, p, nterms):
    terms = []
    for _ in range(nterms):
        nf = rnd.randrange(0, degree + 1)
        facs = tuple(rnd.randrange(k) for _ in range(nf))
        terms.append(Term(rnd.randrange(1, p), facs))
    return terms


def _sc_case(p, fname, tables, terms, degree, claimed, seed, note):
    claim = SumcheckClaim(claimed, [list(t) for t in tables], terms, degree, p)
    tr = Transcript(b"zkl/golden/sumcheck", p, seed)
    start = tr.state
    proof, point = prove_sumcheck(claim, tr)
    return dict(
        field=fname, note=note, state_before=hx(start), claimed_sum=claimed,
        degree=degree, tables=[list(t) for t in tables],
        terms=[[t.coefficient, list(t.factors)] for t in terms],
        rounds=[list(r.evaluations) for r in proof.rounds],
        final_values=list(proof.final_values), point=list(point),
        state_after=hx(tr.state),
    )


def gen_sumcheck():
    cases = []
    rnd = random.Random(99)
    for fname, p in FIELDS.items():
        for trial in range(24):
            n = rnd.randrange(0, 8)
            k = rnd.randrange(1, 8)
            degree = rnd.randrange(1, 4)
            terms = _rand_terms(rnd, k, degree, p, rnd.randrange(1, 6))
            tabs = [[rnd.randrange(p) for _ in range(1 << n)] for _ in range(k)]
            claim = SumcheckClaim(0, tabs, terms, degree, p)
            honest = direct_sum(claim)
            claimed = honest if trial % 4 else (honest + 1) % p
            cases.append(_sc_case(p, fname, tabs, terms, degree, claimed,
                                  b"t%d" % trial, "random"))
        # all-zero factor (test_sumcheck.py:72-79 shape)
        tabs = [[0] * 8, [5, 1, 2, 3, 4, 5, 6, 7]]
        cases.append(_sc_case(p, fname, tabs, [Term(1, (0, 1))], 2, 0, b"z", "zero"))
        # non-canonical entries: negative and >= p, reduced by the prover
        tabs = [[-3, p + 5, 7, -1], [2, 3, 4 * p + 1, 9]]
        terms = [Term(3, (0, 1)), Term(p + 2, (0,))]
        cl = direct_sum(SumcheckClaim(0, tabs, terms, 2, p))
        cases.append(_sc_case(p, fname, tabs, terms, 2, cl, b"nc", "noncanonical"))
        # zero-variable claim
        cases.append(_sc_case(p, fname, [[3], [4]], [Term(1, (0, 1))], 2, 12, b"z0", "n0"))
        # degree-0 term only
        tabs = [[rnd.randrange(p) for _ in range(4)]]
        cases.append(_sc_case(p, fname, tabs, [Term(5, ())], 0, 20 % p, b"d0", "deg0"))
        # larger product-shaped claims (elementprod / lookup shapes)
        for n, shape in ((10, "ep"), (9, "lk")):
            if shape == "ep":
                k, terms, deg = 3, [Term(1, (0, 1, 2))], 3
            else:
                k, deg = 7, 3
                a = rnd.randrange(p)
                terms = [Term(a, (0, 1, 2)), Term((-a) % p, (0, 3)),
                         Term(a * a % p, (0, 4, 5)), Term(a ** 3 % p, (1,)),
                         Term(rnd.randrange(p), (6, 4))]
            tabs = [[rnd.randrange(p) for _ in range(1 << n)] for _ in range(k)]
            cl = direct_sum(SumcheckClaim(0, tabs, terms, deg, p))
            cases.append(_sc_case(p, fname, tabs, terms, deg, cl, b"L" + shape.encode(), shape))
    dump("sumcheck.json", cases)


# ---------------------------------------------------------------------------
def _pt(flat, rv, cv, kind="committed", value=0):
    ref = G.TensorRef(kind, rv, cv, commitment=StubCom(rv + cv) if kind == "committed" else None,
                      value=value)
    return G.ProverTensor(SimpleNamespace(data=list(flat)), ref, ())


def _capture(fn, *args):
    """Run a gadget prover, recording the transcript state right after its
    operand absorption and right after its sumcheck."""
    rec = {}
    orig_abs, orig_sc = G._absorb_operands, G.prove_sumcheck

    def absorb(tr, tag, refs, group):
        rec.setdefault("state_in", tr.state)
        orig_abs(tr, tag, refs, group)
        rec.setdefault("state_before", tr.state)

    def sc(claim, tr):
        rec["state_pre_sumcheck"] = tr.state
        out = orig_sc(claim, tr)
        rec["state_after"] = tr.state
        rec["claimed_sum"] = claim.claimed_sum
        return out

    G._absorb_operands, G.prove_sumcheck = absorb, sc
    try:
        proof = fn(*args)
    finally:
        G._absorb_operands, G.prove_sumcheck = orig_abs, orig_sc
    return proof, rec


def gen_matmul():
    cases = []
    shapes = [
        ("big", (2, 3, 5), None, 11), ("test", (2, 3, 5), None, 12),
        ("test", (4, 4, 1), None, 13), ("test", (1, 1, 1), None, 14),
        ("test", (1, 8, 1), None, 15), ("big", (8, 1, 4), None, 16),
        ("test", (2, 2, 2), (1, 0, 1), 17), ("big", (4, 8, 2), (3, 1, -7), 18),
        ("test", (16, 8, 32), None, 19), ("big", (8, 32, 16), (5, 9, 1), 20),
        ("test", (64, 128, 64), None, 21), ("big", (64, 128, 64), None, 22),
        ("big", (64, 128, 64), (10, 20, 1), 23),
    ]
    for fname, (r, k, c), tamper, seed in shapes:
        p = FIELDS[fname]
        a, b, cm = inputs.matmul_case(seed, r, k, c, tamper=tamper)
        d0, d1, d2 = [(x - 1).bit_length() for x in (a.shape[0], a.shape[1], b.shape[1])]
        ta = _pt(inputs.to_field(a, p), d0, d1)
        tb = _pt(inputs.to_field(b, p), d1, d2)
        tc = _pt(inputs.to_field(cm, p), d0, d2)
        tr = Transcript(b"zkl/golden/matmul", p, b"mm%d" % seed)
        t0 = time.time()
        proof, rec = _capture(G.prove_matmul, ta, tb, tc, KEY, tr, RNG)
        dt = time.time() - t0
        print("matmul", fname, (r, k, c), "dims", (d0, d1, d2), "%.2fs" % dt)
        small = a.size + b.size <= 4096
        cases.append(dict(
            field=fname, shape=[r, k, c], dims=[d0, d1, d2], seed=seed,
            tamper=list(tamper) if tamper else None,
            data=dict(a=a.reshape(-1).tolist(), b=b.reshape(-1).tolist(),
                      c=cm.reshape(-1).tolist()) if small else None,
            state_in=hx(rec["state_in"]), state_before=hx(rec["state_before"]),
            rounds=[list(x.evaluations) for x in proof.sumcheck.rounds],
            final_values=list(proof.sumcheck.final_values),
            state_after=hx(rec["state_after"]),
            openings=[list(o.values) for o in (proof.a_opening, proof.b_opening, proof.c_opening)],
            state_end=hx(tr.state), reference_seconds=dt,
        ))
    dump("matmul.json", cases)


def gen_elementprod():
    cases = []
    for fname, p in FIELDS.items():
        for seed, (r, c) in ((31, (4, 8)), (32, (16, 16)), (33, (1, 2))):
            g = inputs.rng(seed)
            a = g.integers(-300, 300, size=(r, c))
            b = g.integers(-300, 300, size=(r, c))
            cm = a * b
            rv, cv = (r - 1).bit_length(), (c - 1).bit_length()
            ta, tb, tc = (_pt(inputs.to_field(x, p), rv, cv) for x in (a, b, cm))
            tr = Transcript(b"zkl/golden/ep", p, b"ep%d" % seed)
            proof, rec = _capture(G.prove_elementprod, ta, tb, tc, KEY, tr, RNG)
            cases.append(dict(
                field=fname, shape=[r, c], a=a.reshape(-1).tolist(), b=b.reshape(-1).tolist(),
                c=cm.reshape(-1).tolist(), state_in=hx(rec["state_in"]),
                state_before=hx(rec["state_before"]),
                state_pre_sumcheck=hx(rec["state_pre_sumcheck"]),
                claimed_sum=rec["claimed_sum"],
                rounds=[list(x.evaluations) for x in proof.sumcheck.rounds],
                final_values=list(proof.sumcheck.final_values),
                state_after=hx(rec["state_after"]),
                ab_opening=list(proof.ab_opening.values), state_end=hx(tr.state),
            ))
    dump("elementprod.json", cases)


# ---------------------------------------------------------------------------
def _lookup_case(fname, secret, table, mult, seed, note):
    p = FIELDS[fname]
    lt = L.LookupTable(tuple(table), StubCom((len(table) - 1).bit_length()), "t")
    sv = L.SecretVector(tuple(secret), StubCom((len(secret) - 1).bit_length()), ())
    tr = Transcript(b"zkl/golden/lookup", p, seed)
    start = tr.state
    rec = {}
    orig_sc = L.prove_sumcheck

    def sc(claim, t):
        rec["state_pre_sumcheck"] = t.state
        out = orig_sc(claim, t)
        rec["state_after"] = t.state
        return out

    L.prove_sumcheck = sc
    try:
        pr = L.prove_lookup(sv, list(mult), lt, KEY, tr, RNG)
    finally:
        L.prove_sumcheck = orig_sc
    return dict(
        field=fname, note=note, secret=list(secret), table=list(table), mult=list(mult),
        state_before=hx(start), secret_vars=pr.secret_vars, beta_retries=pr.beta_retries,
        rounds=[list(x.evaluations) for x in pr.sumcheck.rounds],
        final_values=list(pr.sumcheck.final_values),
        secret_values=list(pr.secret_values), table_values=list(pr.table_values),
        state_pre_sumcheck=hx(rec["state_pre_sumcheck"]), state_after=hx(rec["state_after"]),
        state_end=hx(tr.state),
    )


def gen_lookup():
    cases, mcases = [], []
    rnd = random.Random(77)
    for fname, p in FIELDS.items():
        specs = []
        t = [rnd.randrange(1, 1 << 16) for _ in range(32)]
        specs.append(("d<n", [rnd.choice(t) for _ in range(4)], t))
        t = [rnd.randrange(1, 1 << 16) for _ in range(4)]
        specs.append(("d>n", [rnd.choice(t) for _ in range(32)], t))
        specs.append(("d=n", [100, 107, 103, 103, 100, 101, 106, 105], list(range(100, 108))))
        specs.append(("single", [57], list(range(50, 66))))
        specs.append(("dup", [7] * 16, list(range(16))))
        t = [rnd.randrange(p) for _ in range(64)]
        specs.append(("big-d", [rnd.choice(t) for _ in range(1024)], t))
        t = [rnd.randrange(p) for _ in range(1024)]
        specs.append(("big-n", [rnd.choice(t) for _ in range(64)], t))
        t = [5, 9, 5, 11]  # duplicate table value: last index wins (lookup.py:92)
        specs.append(("table-dup", [5, 9, 11, 5, 5, 9, 11, 11], t))
        for note, sec, tab in specs:
            m = L.compute_multiplicities(sec, L.LookupTable(tuple(tab), None))
            cases.append(_lookup_case(fname, sec, tab, m, note.encode(), note))
        # forced wrong multiplicities -> proof exists, verifier must reject
        cases.append(_lookup_case(fname, [1, 2, 3, 99], list(range(8)),
                                  [0, 1, 1, 1, 1, 0, 0, 0], b"oot", "out-of-table"))
        m = L.compute_multiplicities([1, 2, 3, 4], L.LookupTable(tuple(range(8)), None))
        m[1], m[5] = m[5], m[1]
        cases.append(_lookup_case(fname, [1, 2, 3, 4], list(range(8)), m, b"wm", "wrong-mult"))
        # multiplicity known answers
        for sec, tab in (([20, 20, 40, 10], [10, 20, 30, 40]), ([20, 99], [10, 20, 30, 40]),
                         ([5, 5, 7, 1], [5, 1, 7, 5]), ([3, 4, 8], [3, 4, 5, 6])):
            try:
                out = dict(counts=L.compute_multiplicities(sec, L.LookupTable(tuple(tab), None)))
            except L.ElementNotInTable as e:
                out = dict(error=[e.index, e.value])
            mcases.append(dict(field=fname, secret=sec, table=tab, **out))
    dump("lookup.json", dict(lookup=cases, multiplicities=mcases))


def gen_pair_lookup():
    """SiLU pair lookup (gadgets.py:679-688) on a small table, both fields."""
    cases = []
    params = QuantParams(gamma_fp=2**4, bound=2**6, zeta=2**4, xi=2**9,
                         radices=(8, 8, 8), act_bound=4)
    for fname, p in FIELDS.items():
        xs, ys = TB.silu_entries(params)
        xcol = tuple(x % p for x in xs)
        ycol = tuple(y % p for y in ys)
        pair = TB.PairTable(L.LookupTable(xcol, StubCom(7)), L.LookupTable(ycol, StubCom(7)), "silu")
        g = inputs.rng(5)
        q = g.integers(xs[0], xs[-1] + 1, size=256)
        out = [TB.silu_value(params, int(v)) for v in q]
        xt = _pt([int(v) % p for v in q], 4, 4)
        yt = _pt([int(v) % p for v in out], 4, 4)
        tr = Transcript(b"zkl/golden/pair", p, b"pair")
        start = tr.state
        pr = G._prove_pair_lookup(b"swiglu/act", xt, yt, pair, KEY, tr, RNG)
        cases.append(dict(
            field=fname, x=[int(v) for v in q], y=out, table_x=list(xs), table_y=list(ys),
            state_before=hx(start), beta_retries=pr.beta_retries,
            rounds=[list(x.evaluations) for x in pr.sumcheck.rounds],
            final_values=list(pr.sumcheck.final_values),
            secret_values=list(pr.secret_values), table_values=list(pr.table_values),
            state_end=hx(tr.state),
        ))
    dump("pair_lookup.json", cases)


def gen_tables():
    params = QuantParams(gamma_fp=2**12, bound=2**16, zeta=2**12, xi=2**64,
                         radices=(2**16,) * 4, act_bound=8)
    out = {}
    fns = (("silu", TB.silu_entries), ("silu_deriv", TB.silu_deriv_entries),
           ("exp0", lambda q: TB.exp_segment_entries(q, 0)),
           ("rsqrt_eps1e-5", lambda q: TB.rsqrt_entries(q, 1e-5)))
    # the LLaMA block's tables (paper_2508_21393_b200/block.py): SiLU / SiLU'
    # at gamma/2 = 2^11 with act_bound 16, and the exp segment of base 4
    half = QuantParams(gamma_fp=2**11, bound=2**16, zeta=2**11, xi=2**64,
                       radices=(2**16,) * 4, act_bound=16)
    base4 = QuantParams(gamma_fp=2**12, bound=2**16, zeta=2**12, xi=2**18,
                        radices=(4, 2**16), act_bound=8)
    fns += (("silu_g2048_a16", lambda q: TB.silu_entries(half)),
            ("silu_deriv_g2048_a16", lambda q: TB.silu_deriv_entries(half)),
            ("exp_base4", lambda q: TB.exp_segment_entries(base4, 1)))
    for name, fn in fns:
        xs, ys = fn(params)
        arr = np.asarray(ys, dtype="<i4")
        out[name] = dict(x0=xs[0], n=len(xs),
                         y_zlib_b64=base64.b64encode(zlib.compress(arr.tobytes(), 9)).decode())
    dump("tables_g4096.json", out)


def gen_field_mle():
    rnd = random.Random(5)
    out = dict(batch_inverse=[], eq=[], fold=[], mle=[])
    for fname, p in FIELDS.items():
        for n in (1, 2, 7, 64, 300):
            v = [rnd.randrange(1, p) for _ in range(n)]
            out["batch_inverse"].append(dict(field=fname, values=v, inverse=F.batch_inverse(v, p)))
        v = [rnd.randrange(1, p) for _ in range(10)]
        v[6] = 0
        v[8] = 0
        try:
            F.batch_inverse(v, p)
        except F.InversionOfZero as e:
            out["batch_inverse"].append(dict(field=fname, values=v, error=str(e)))
        for m in (0, 1, 3, 6):
            pt = [rnd.randrange(p) for _ in range(m)]
            out["eq"].append(dict(field=fname, point=pt, table=M.eq_table(pt, p)))
        for m in (1, 4):
            t = [rnd.randrange(p) for _ in range(1 << m)]
            r = rnd.randrange(p)
            out["fold"].append(dict(field=fname, table=t, r=r, out=M.fold_table(t, r, p)))
            pt = [rnd.randrange(p) for _ in range(m)]
            out["mle"].append(dict(field=fname, table=t, point=pt, value=M.mle_evaluate(t, pt, p)))
    dump("field_mle.json", out)


def _lookup_rec(lp):
    return dict(beta_retries=lp.beta_retries,
                rounds=[list(x.evaluations) for x in lp.sumcheck.rounds],
                final_values=list(lp.sumcheck.final_values),
                secret_values=list(lp.secret_values), table_values=list(lp.table_values))


def gen_nonlinear():
    """prove_rescale / prove_swiglu (phi, phi_prime) / prove_rsqrt
    (gadgets.py:585-622, 761-771, 842-847) on 16x16 tensors, both fields."""
    from zklora.quantize import centered_divmod

    params = QuantParams(gamma_fp=2**4, bound=2**6, zeta=2**4, xi=2**9,
                         radices=(8, 8, 8), act_bound=4)
    eps = 2.0 ** -6
    half = params.act_bound * params.gamma_fp
    cases = []
    for fname, p in FIELDS.items():
        # build_table_set's params_digest packs the modulus into 16 bytes
        # (tables.py:192), which overflows for BLS12-381 Fr: assemble the same
        # TableSet fields directly (tables.py:217-238)
        ts = TB.TableSet(
            params, eps, p, b"", (),
            TB._pair("silu", TB.silu_entries(params), KEY, p),
            TB._pair("silu_deriv", TB.silu_deriv_entries(params), KEY, p),
            TB._pair("rsqrt", TB.rsqrt_entries(params, eps), KEY, p),
            L.make_lookup_table(TB._encode_column(TB.quant_range_entries(params), p), KEY,
                                "quant_range"),
            L.make_lookup_table(TB._encode_column(TB.residue_range_entries(params), p), KEY,
                                "residue_range"))
        g = inputs.rng(11)
        enc = lambda vals: [int(v) % p for v in vals]
        # rescale, divisor = zeta (lift 1) and divisor = zeta/4 (lift 4)
        for divisor in (params.zeta, params.zeta // 4):
            lift = params.zeta // divisor
            q0 = g.integers(-half, half, size=256)
            r0 = g.integers(-(divisor // 2), divisor // 2, size=256)
            wide = [int(divisor * a + b) for a, b in zip(q0, r0)]
            qr = [centered_divmod(w, divisor) for w in wide]
            narrow = [q for q, _ in qr]
            resid = [r * lift for _, r in qr]
            tr = Transcript(b"zkl/golden/rescale", p, b"d%d" % divisor)
            start = tr.state
            pr = G.prove_rescale(_pt(enc(wide), 4, 4), _pt(enc(narrow), 4, 4),
                                 _pt(enc(resid), 4, 4), divisor, ts, KEY, tr, RNG)
            cases.append(dict(gadget="rescale", field=fname, divisor=divisor, wide=wide,
                              narrow=narrow, resid=resid, state_before=hx(start),
                              identity=list(pr.identity_opening.values),
                              lookups=[_lookup_rec(pr.quant_lookup), _lookup_rec(pr.resid_lookup)],
                              state_end=hx(tr.state)))
        for mode in ("phi", "phi_prime"):
            fn = TB.silu_value if mode == "phi" else TB.silu_deriv_value
            q0 = g.integers(-half, half, size=256)
            r0 = g.integers(-(params.zeta // 2), params.zeta // 2, size=256)
            wide = [int(params.zeta * a + b) for a, b in zip(q0, r0)]
            qr = [centered_divmod(w, params.zeta) for w in wide]
            narrow = [q for q, _ in qr]
            resid = [r for _, r in qr]
            out = [fn(params, q) for q in narrow]
            tr = Transcript(b"zkl/golden/swiglu", p, mode.encode())
            start = tr.state
            pr = G.prove_swiglu(_pt(enc(wide), 4, 4), _pt(enc(out), 4, 4), _pt(enc(narrow), 4, 4),
                                _pt(enc(resid), 4, 4), mode, ts, KEY, tr, RNG)
            cases.append(dict(gadget="swiglu", mode=mode, field=fname, wide=wide, narrow=narrow,
                              resid=resid, out=out, state_before=hx(start),
                              identity=list(pr.identity_opening.values),
                              lookups=[_lookup_rec(pr.activation_lookup),
                                       _lookup_rec(pr.resid_lookup)],
                              state_end=hx(tr.state)))
        v = [int(x) for x in g.integers(0, half, size=64)]
        u = [TB.rsqrt_value(params, eps, x) for x in v]
        tr = Transcript(b"zkl/golden/rsqrt", p, b"r")
        start = tr.state
        pr = G.prove_rsqrt(_pt(enc(v), 3, 3), _pt(enc(u), 3, 3), ts, KEY, tr, RNG)
        cases.append(dict(gadget="rsqrt", field=fname, v=v, u=u, state_before=hx(start),
                          lookups=[_lookup_rec(pr.lookup)], state_end=hx(tr.state)))
    tabs = {}
    for name in ("silu", "silu_deriv", "rsqrt"):
        pt_ = getattr(ts, name)
        tabs[name] = dict(x=[F.to_signed(v, p) for v in pt_.x.entries],
                          y=[F.to_signed(v, p) for v in pt_.y.entries])
    tabs["quant_range"] = [F.to_signed(v, p) for v in ts.quant_range.entries]
    tabs["residue_range"] = [F.to_signed(v, p) for v in ts.residue_range.entries]
    dump("nonlinear.json", dict(params=dict(gamma=16, zeta=16, act_bound=4, eps=eps),
                                tables=tabs, cases=cases))


class RefBlockProver:
    """Drives the REFERENCE's gadget provers (stub commitments) through
    paper_2508_21393_b200.block.prove_block's schedule on CPU tensors, so the
    GPU block proof can be checked byte for byte (tests/test_gpu_block.py)."""

    def __init__(self, tr, ts, fp, p):
        import torch
        from paper_2508_21393_b200 import block as BK

        self.BK, self.torch = BK, torch
        self.tr, self.ts, self.fp, self.p = tr, ts, fp, p
        ys = lambda pair: torch.tensor([F.to_signed(v, p) for v in pair.y.entries],  # noqa: E731
                                       dtype=torch.int32)
        self.luts = {"silu": ys(ts.silu), "silu_deriv": ys(ts.silu_deriv),
                     "rsqrt": ys(ts.rsqrt), "exp": ys(ts.exp_segments[0]),
                     "act_x0": F.to_signed(ts.silu.x.entries[0], p)}
        self.log = []

    def pt(self, t):
        rv, cv = (t.shape[0] - 1).bit_length(), (t.shape[1] - 1).bit_length()
        return _pt([int(v) % self.p for v in t.reshape(-1).tolist()], rv, cv)

    def matmul(self, a, b, c):
        pr = G.prove_matmul(self.pt(a), self.pt(b), self.pt(c), KEY, self.tr, RNG)
        self.log.append(["matmul", len(pr.sumcheck.rounds)])

    def matadd(self, a, b, c, sign):
        G.prove_matadd(self.pt(a), self.pt(b), self.pt(c), sign, KEY, self.tr, RNG)
        self.log.append(["matadd"])

    def eprod(self, a, b, c):
        pr = G.prove_elementprod(self.pt(a), self.pt(b), self.pt(c), KEY, self.tr, RNG)
        self.log.append(["elementprod", len(pr.sumcheck.rounds)])

    def rescale(self, wide, divisor):
        q, r = self.BK._divmod(wide, divisor, self.fp)
        pr = G.prove_rescale(self.pt(wide), self.pt(q), self.pt(r), divisor, self.ts, KEY,
                             self.tr, RNG)
        self.log.append(["rescale", len(pr.quant_lookup.sumcheck.rounds),
                         len(pr.resid_lookup.sumcheck.rounds)])
        return q

    def swiglu(self, wide, mode):
        q, r = self.BK._divmod(wide, self.fp.zeta, self.fp)
        out = self.BK._lut(self.luts["silu" if mode == "phi" else "silu_deriv"], q,
                           self.luts["act_x0"]).to(self.torch.int16)
        pr = G.prove_swiglu(self.pt(wide), self.pt(out), self.pt(q), self.pt(r), mode, self.ts,
                            KEY, self.tr, RNG)
        self.log.append(["swiglu", len(pr.activation_lookup.sumcheck.rounds),
                         len(pr.resid_lookup.sumcheck.rounds)])
        return out

    def rsqrt(self, v, u):
        pr = G.prove_rsqrt(self.pt(v), self.pt(u), self.ts, KEY, self.tr, RNG)
        self.log.append(["rsqrt", len(pr.lookup.sumcheck.rounds)])

    def exp_lookup(self, v, e):
        pr = G._prove_pair_lookup(b"softmax/exp0", self.pt(v), self.pt(e), self.ts.exp_segments[0],
                                  KEY, self.tr, RNG)
        self.log.append(["softmax_exp", len(pr.sumcheck.rounds)])


TINY_BLOCK = dict(shape=("tiny", 16, 16, 2, 8, 24, 2, ("q", "v", "o")),
                  fp=dict(gamma_fp=16, zeta=16, act_bound=4, exp_n=64, eps=2.0 ** -6,
                          exp_base=4, act_shift=1, eta_div=8),
                  wstd=0.2, dy_std=0.3)


def gen_block():
    """A tiny LoRA block (2 heads, FFN padded 24 -> 32, LoRA on q, v, o) proven
    by the reference's gadgets in prove_block's order, test field and big
    field; the end transcript state pins the whole composition.  The tables are
    the reference's own table functions (tables.py) at the block's scales:
    exp segment of radices (exp_base, exp_n), SiLU / SiLU' at gamma/2."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2508_21393_b200 import block as BK

    shape = BK.BlockShape(*TINY_BLOCK["shape"])
    fp = BK.FixedPoint(**TINY_BLOCK["fp"])
    g, a = fp.gamma_fp, fp.act_bound
    params = QuantParams(gamma_fp=g, bound=2**6, zeta=fp.zeta, xi=2**9, radices=(64, 8),
                         act_bound=a)
    pexp = QuantParams(gamma_fp=g, bound=2**6, zeta=fp.zeta, xi=2**8,
                       radices=(fp.exp_base, fp.exp_n), act_bound=a)
    ga, aa = g >> fp.act_shift, a << fp.act_shift
    pact = QuantParams(gamma_fp=ga, bound=2**6, zeta=ga, xi=2**9, radices=(64, 8),
                       act_bound=aa)
    cases = []
    for fname, p in FIELDS.items():
        ts = TB.TableSet(
            params, fp.eps, p, b"", (TB._pair("exp0", TB.exp_segment_entries(pexp, 1), KEY, p),),
            TB._pair("silu", TB.silu_entries(pact), KEY, p),
            TB._pair("silu_deriv", TB.silu_deriv_entries(pact), KEY, p),
            TB._pair("rsqrt", TB.rsqrt_entries(params, fp.eps), KEY, p),
            L.make_lookup_table(TB._encode_column(TB.quant_range_entries(params), p), KEY,
                                "quant_range"),
            L.make_lookup_table(TB._encode_column(TB.residue_range_entries(params), p), KEY,
                                "residue_range"))
        w = BK.BlockWitness(shape, seed=3, fp=fp, device="cpu", wstd=TINY_BLOCK["wstd"],
                            dy_std=TINY_BLOCK["dy_std"])
        tr = Transcript(b"zkl/golden/block", p, fname.encode())
        start = tr.state
        t0 = time.time()
        P = BK.prove_block(w, RefBlockProver(tr, ts, fp, p))
        print("block", fname, "%.1f s" % (time.time() - t0), len(P.log), "gadgets")
        cases.append(dict(field=fname, seed=3, state_before=hx(start), log=P.log,
                          state_end=hx(tr.state)))
    dump("block.json", dict(shape=list(TINY_BLOCK["shape"][1:7]) + [list(TINY_BLOCK["shape"][7])],
                            fp=TINY_BLOCK["fp"], wstd=TINY_BLOCK["wstd"],
                            dy_std=TINY_BLOCK["dy_std"], cases=cases))


def gen_softmax():
    """prove_softmax_row (gadgets.py:930-1036) on 8- and 16-entry rows at the
    reference tests' DESK parameters, both fields."""
    params = QuantParams(gamma_fp=2**7, bound=2**11, zeta=2**7, xi=2**21,
                         radices=(2**7, 2**7, 2**7), act_bound=16)
    eps = 1e-5
    g = params.gamma_fp
    cases = []
    tabs = None
    for fname, p in FIELDS.items():
        exps = tuple(TB._pair("exp%d" % k, TB.exp_segment_entries(params, k), KEY, p)
                     for k in range(params.num_radices))
        ts = TB.TableSet(
            params, eps, p, b"", exps,
            TB._pair("silu", TB.silu_entries(params), KEY, p),
            TB._pair("silu_deriv", TB.silu_deriv_entries(params), KEY, p),
            TB._pair("rsqrt", TB.rsqrt_entries(params, eps), KEY, p),
            L.make_lookup_table(TB._encode_column(TB.quant_range_entries(params), p), KEY,
                                "quant_range"),
            L.make_lookup_table(TB._encode_column(TB.residue_range_entries(params), p), KEY,
                                "residue_range"))
        if tabs is None:
            tabs = dict(exp=[[F.to_signed(v, p) for v in e.y.entries] for e in exps],
                        quant_range=[F.to_signed(v, p) for v in ts.quant_range.entries],
                        residue_range=[F.to_signed(v, p) for v in ts.residue_range.entries])
        rnd = random.Random(92)
        for row_len in (8, 16):
            zs = [rnd.randint(-3 * g, 3 * g) for _ in range(row_len)]
            wit = G.softmax_row_witness(zs, params, p)
            n = (row_len - 1).bit_length()
            z_t = _pt([z % p for z in zs], 0, n)
            p_t = _pt([v % p for v in wit[4]], 0, n)
            tr = Transcript(b"zkl/golden/softmax", p, b"%d" % row_len)
            start = tr.state
            pr = G.prove_softmax_row(z_t, p_t, wit, ts, KEY, tr, RNG)
            cases.append(dict(
                field=fname, z=zs, xi_prime=wit[0], digits=wit[1], partials=wit[2],
                chain=[[list(w), list(q), list(r)] for w, q, r in wit[3]], p=list(wit[4]),
                state_before=hx(start),
                decomposition=list(pr.decomposition_opening.values),
                digit_lookups=[_lookup_rec(x) for x in pr.digit_lookups],
                chain_prods=[[list(r.evaluations) for r in x.sumcheck.rounds]
                             for x in pr.chain_prod_proofs],
                chain_rescales=[[_lookup_rec(x.quant_lookup), _lookup_rec(x.resid_lookup)]
                                for x in pr.chain_rescale_proofs],
                normalization=list(pr.normalization_opening.values),
                state_end=hx(tr.state)))
    dump("softmax.json", dict(params=dict(gamma=g, zeta=params.zeta, act_bound=16,
                                          radices=list(params.radices), xi=params.xi),
                              tables=tabs, cases=cases))


if __name__ == "__main__":
    which = sys.argv[1:] or ["transcript", "sumcheck", "matmul", "elementprod", "lookup",
                             "pair_lookup", "tables", "field_mle", "nonlinear", "block", "softmax"]
    for w in which:
        globals()["gen_" + w]()
