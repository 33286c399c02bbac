"""GPU parity of the non-linear gadget mirrors (rescale, SwiGLU, rsqrt) and of
device MLE evaluation of integer matrices.

The goldens (tests/golden/nonlinear.json) come from the reference's own
prove_rescale / prove_swiglu / prove_rsqrt (gadgets.py:600-622, 761-782,
842-847) run with the stub commitment; tests/test_oracle_golden.py pins the
oracle restatement to the same file."""

from types import SimpleNamespace

import pytest

from conftest import FIELDS, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2508_21393_b200 as zb  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402
from paper_2508_21393_b200 import mle as M  # noqa: E402
from paper_2508_21393_b200 import nonlinear as NL  # noqa: E402
from paper_2508_21393_b200.commit_stub import StubCommitment, StubKey  # noqa: E402
from paper_2508_21393_b200.gadgets import DeviceMatrix, ProverTensor, TensorRef  # noqa: E402
from paper_2508_21393_b200.transcript import Transcript  # noqa: E402

KEY = StubKey()


class _Rng:
    def vector(self, n):
        return [0] * n


def _log2(n):
    return (n - 1).bit_length()


def _tables(g, p, where):
    t = g["tables"]
    spec = D.spec_for(p)
    enc = lambda vals: tuple(v % p for v in vals)  # noqa: E731

    def rng_table(vals, name):
        c = StubCommitment(_log2(len(vals)))
        if where == "device":
            return NL.device_range_table(vals[0], len(vals), spec, c, name)
        return zb.LookupTable(enc(vals), c, name)

    def pair(name):
        xs, ys = t[name]["x"], t[name]["y"]
        c = StubCommitment(_log2(len(xs)))
        if where == "device":
            return NL.device_pair_table(xs, ys, c, c, name)
        return NL.PairTable(zb.LookupTable(enc(xs), c, name + ".x"),
                            zb.LookupTable(enc(ys), c, name + ".y"), name)

    return NL.TableSet(SimpleNamespace(zeta=g["params"]["zeta"]), g["params"]["eps"], p, b"", (),
                       pair("silu"), pair("silu_deriv"), pair("rsqrt"),
                       rng_table(t["quant_range"], "quant_range"),
                       rng_table(t["residue_range"], "residue_range"))


def _operand(vals, rv, cv, p, where, dtype=torch.int32):
    ref = TensorRef("committed", rv, cv, commitment=StubCommitment(rv + cv))
    if vals is None:
        return ProverTensor(None, ref, ())
    if where == "device":
        t = torch.tensor(vals, dtype=dtype).cuda().view(1 << rv, 1 << cv)
        return ProverTensor(None, ref, (), device=DeviceMatrix.from_int_tensor(t))
    return ProverTensor(SimpleNamespace(data=[v % p for v in vals]), ref, ())


def _check_lookup(got, want):
    assert got.beta_retries == want["beta_retries"]
    assert [list(r.evaluations) for r in got.sumcheck.rounds] == want["rounds"]
    assert list(got.sumcheck.final_values) == want["final_values"]
    assert list(got.secret_values) == want["secret_values"]
    assert list(got.table_values) == want["table_values"]


@pytest.mark.parametrize("where", ["device", "host"])
def test_nonlinear_golden(where):
    g = load_golden("nonlinear.json")
    seen = set()
    for c in g["cases"]:
        p = FIELDS[c["field"]]
        ts = _tables(g, p, where)
        tr = Transcript.from_state(bytes.fromhex(c["state_before"]), p)
        op = lambda vals, k=4: _operand(vals, k, k, p, where)  # noqa: E731
        if c["gadget"] == "rescale":
            pr = zb.prove_rescale(op(c["wide"]), op(c["narrow"]), op(c["resid"]), c["divisor"], ts,
                                  KEY, tr, _Rng())
            assert pr.divisor == c["divisor"] and pr.shape == (4, 4)
            lookups = [pr.quant_lookup, pr.resid_lookup]
        elif c["gadget"] == "swiglu":
            pr = zb.prove_swiglu(op(c["wide"]), op(c["out"]), op(c["narrow"]), op(c["resid"]),
                                 c["mode"], ts, KEY, tr, _Rng())
            assert pr.mode == c["mode"]
            lookups = [pr.activation_lookup, pr.resid_lookup]
        else:
            pr = zb.prove_rsqrt(op(c["v"], 3), op(c["u"], 3), ts, KEY, tr, _Rng())
            lookups = [pr.lookup]
        if "identity" in c:
            assert list(pr.identity_opening.values) == c["identity"]
        for got, want in zip(lookups, c["lookups"]):
            _check_lookup(got, want)
        assert tr.state.hex() == c["state_end"], (c["gadget"], c["field"])
        seen.add((c["gadget"], c["field"]))
    assert len(seen) == 6


def test_rescale_errors_like_reference():
    g = load_golden("nonlinear.json")
    p = FIELDS["test"]
    ts = _tables(g, p, "device")
    c = [c for c in g["cases"] if c["gadget"] == "rescale"][0]
    op = lambda vals, k=4: _operand(vals, k, k, p, "device")  # noqa: E731
    with pytest.raises(ValueError):
        zb.prove_rescale(op(c["wide"]), op(c["narrow"]), op(c["resid"]), 3, ts, KEY,
                         Transcript(b"x", p, b""), _Rng())
    with pytest.raises(zb.ShapeMismatch):
        zb.prove_rescale(op(c["wide"]), op(c["narrow"][:64], 3), op(c["resid"]), 16, ts, KEY,
                         Transcript(b"x", p, b""), _Rng())
    # a quotient outside quant_range: ElementNotInTable at the first bad index
    bad = list(c["narrow"])
    bad[37] = 1000
    bad[90] = -1000
    with pytest.raises(zb.ElementNotInTable) as e:
        zb.prove_rescale(op(c["wide"]), op(bad), op(c["resid"]), 16, ts, KEY,
                         Transcript(b"x", p, b""), _Rng())
    assert e.value.index == 37


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("shape", [(0, 0), (0, 5), (5, 0), (3, 4), (7, 6)])
@pytest.mark.parametrize("dtype", [torch.int16, torch.int32, torch.int64])
def test_mle_of_int_matrix(field, shape, dtype):
    """mle_evaluate_matrix (one integer matvec) == the lifted-vector fold."""
    import random

    p = FIELDS[field]
    spec = D.spec_for(p)
    rv, cv = shape
    gen = torch.Generator().manual_seed(rv * 16 + cv)
    hi = {torch.int16: 1 << 15, torch.int32: 1 << 31, torch.int64: 1 << 62}[dtype]
    t = torch.randint(-hi, hi, (1 << rv, 1 << cv), generator=gen, dtype=torch.int64).to(dtype)
    rnd = random.Random(rv + cv)
    pt = [rnd.randrange(p) for _ in range(rv + cv)]
    Mx = DeviceMatrix.from_int_tensor(t.cuda())
    got = M.mle_evaluate_any(Mx, pt, p)
    want = M.mle_evaluate([int(v) % p for v in t.reshape(-1).tolist()], pt, p)
    assert got == want


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("dims", [(0, 3, 2), (2, 0, 3), (3, 4, 3), (6, 7, 6)])
def test_replicated_dense_matmul_matches_factored_and_oracle(field, dims):
    """The reference's materialised zkMat claim on the dense engine, the
    factored prover and the oracle's dense restatement agree bit for bit."""
    import numpy as np

    from oracle import fs, zkmat
    from paper_2508_21393_b200.gadgets import matmul_sumcheck, matmul_sumcheck_replicated

    p = FIELDS[field]
    d0, d1, d2 = dims
    g = np.random.Generator(np.random.PCG64(sum(dims)))
    a = g.integers(-32768, 32768, (1 << d0, 1 << d1)).astype(np.int16)
    b = g.integers(-32768, 32768, (1 << d1, 1 << d2)).astype(np.int16)
    c = a.astype(np.int64) @ b.astype(np.int64)
    c[0, 0] += 1  # a false claim: g(1) must still be computed, not derived
    mats = [DeviceMatrix.from_int_tensor(torch.from_numpy(x).cuda()) for x in (a, b, c)]
    t1, t2 = Transcript(b"rep", p, b"s"), Transcript(b"rep", p, b"s")
    r1 = matmul_sumcheck_replicated(*mats, dims, t1)
    mats = [DeviceMatrix.from_int_tensor(torch.from_numpy(x).cuda()) for x in (a, b, c)]
    r2 = matmul_sumcheck(*mats, dims, t2)
    assert [tuple(x) for x in r1[0]] == [tuple(x) for x in r2[0]]
    assert list(r1[1]) == list(r2[1]) and tuple(r1[2]) == tuple(r2[2])
    assert t1.state == t2.state
    t3 = fs.FS(b"rep", p, b"s")
    A = [int(v) % p for v in a.reshape(-1)]
    B = [int(v) % p for v in b.reshape(-1)]
    C = [int(v) % p for v in c.reshape(-1)]
    out = zkmat.prove_dense(A, B, C, dims, t3)
    assert [list(x) for x in r1[0]] == [list(x) for x in out[0]]
    assert t3.state == t1.state


@pytest.mark.parametrize("n", [16, 4096, 1 << 16])
@pytest.mark.parametrize("dtype", [torch.int16, torch.int32, torch.int64])
def test_range_multiplicities_vs_bincount(n, dtype):
    """zkl_range_multiplicities (shared-memory bins for n <= 12288, warp-merged
    global atomics above) against torch.bincount, skewed inputs included."""
    from paper_2508_21393_b200 import lookup as L

    p = FIELDS["big"]
    spec = D.spec_for(p)
    lo = -(n // 2)
    tab = NL.device_range_table(lo, n, spec, StubCommitment(_log2(n)), "r")
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randint(lo, lo + n, (1 << 20,), device="cuda", generator=g, dtype=torch.int64)
    x[: 1 << 18] = lo + n // 3  # one hot bin (padding-like skew)
    col = x.to(dtype)
    sec = D.LiftedColumn(col, spec)
    counts, index = L.multiplicities_range(sec, tab, col, tab.int_column)
    want = torch.bincount((x - lo).long(), minlength=n)
    got = torch.tensor(D.download(counts.buf, spec, n), dtype=torch.int64)
    assert torch.equal(got, want.cpu())
    assert torch.equal(index[: x.numel()].long(), (x - lo).long())
    assert sec._buf is None  # never lifted
    if dtype == torch.int16 and n == 1 << 16:
        return  # every int16 is in the table
    bad = col.clone()
    bad[777] = lo + n
    bad[900] = lo - 1
    with pytest.raises(zb.ElementNotInTable) as e:
        L.multiplicities_range(D.LiftedColumn(bad, spec), tab, bad, tab.int_column)
    assert e.value.index == 777 and e.value.value == int(bad[777]) % p


@pytest.mark.parametrize("divisor", [4096, 1024, 1])
@pytest.mark.parametrize("dtype", [torch.int64, torch.int32, torch.int16])
def test_rescale_witness_device_vs_reference_divmod(divisor, dtype):
    """zkl_rescale_witness == centered_divmod (quantize.py:101-104) entry for
    entry; out-of-domain quotients raise RangeViolation (nothing is clamped)."""
    fp = SimpleNamespace(zeta=4096, gamma_fp=4096, act_bound=8)
    g = torch.Generator().manual_seed(divisor)
    hi = {torch.int64: 1 << 27, torch.int32: 1 << 27, torch.int16: 1 << 15}[dtype]
    w = torch.randint(-hi, hi, (1 << 16,), generator=g, dtype=torch.int64)
    w = w.clamp(-32768 * divisor + 1, 32767 * divisor - 1).to(dtype)
    q, r = NL.rescale_witness_device(w.cuda(), divisor, fp)
    wl = w.tolist()
    for i in range(0, len(wl), 997):
        qq = (wl[i] + divisor // 2) // divisor
        assert int(q[i]) == qq and int(r[i]) == (wl[i] - divisor * qq) * (4096 // divisor)
    if dtype == torch.int16 and divisor == 1:
        return
    big = w.clone().to(torch.int64)
    big[123] = 40000 * divisor
    big[456] = -40000 * divisor
    with pytest.raises(NL.RangeViolation, match=r"\(2 entries\)"):
        NL.rescale_witness_device(big.cuda(), divisor, fp)


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("n", [6, 9, 13, 21])
def test_eq_factored_elementprod_matches_dense(field, n, monkeypatch):
    """prove_elementprod's eq-factored path (tiled logUp engine with term
    coefficients (1,0,0,0,0)) gives the dense engine's proof byte for byte."""
    from paper_2508_21393_b200 import gadgets as G

    p = FIELDS[field]
    g = torch.Generator().manual_seed(n)
    rv = n // 2
    a = torch.randint(-32768, 32768, (1 << rv, 1 << (n - rv)), generator=g).short()
    b = torch.randint(-32768, 32768, (1 << rv, 1 << (n - rv)), generator=g).short()
    c = a.long() * b.long()
    c[0, 1] += 5  # a false claim too: every evaluation is computed, not derived

    def run(factored):
        monkeypatch.setattr(G, "EQ_FACTORED_MIN_VARS", 6 if factored else 99)
        monkeypatch.setattr(G, "EQ_TILE_LOG", 5 if n < 21 else 16)
        tr = Transcript(b"ep", p, b"s")
        ops = [_operand(None, rv, n - rv, p, "device") for _ in range(3)]
        ops = [ProverTensor(None, o.ref, (), device=DeviceMatrix.from_int_tensor(t.cuda()))
               for o, t in zip(ops, (a, b, c))]
        pr = zb.prove_elementprod(*ops, KEY, tr, _Rng())
        return pr, tr.state

    p1, s1 = run(True)
    p2, s2 = run(False)
    assert [tuple(r.evaluations) for r in p1.sumcheck.rounds] == \
        [tuple(r.evaluations) for r in p2.sumcheck.rounds]
    assert tuple(p1.sumcheck.final_values) == tuple(p2.sumcheck.final_values)
    assert s1 == s2


@pytest.mark.parametrize("where", ["device", "host"])
def test_softmax_row_golden(where):
    """prove_softmax_row (gadgets.py:930-1036) bit-exact with the reference's
    own run: decomposition and normalisation openings, the three exp digit
    pair lookups, the chain's elementprods and rescales, the end state."""
    g = load_golden("softmax.json")
    prm = g["params"]
    params = SimpleNamespace(gamma_fp=prm["gamma"], zeta=prm["zeta"], xi=prm["xi"],
                             radices=tuple(prm["radices"]), act_bound=prm["act_bound"])
    for c in g["cases"]:
        p = FIELDS[c["field"]]
        spec = D.spec_for(p)
        t = g["tables"]
        enc = lambda vals: tuple(v % p for v in vals)  # noqa: E731

        def pair(k):
            ys = t["exp"][k]
            xs = list(range(len(ys)))
            com = StubCommitment(_log2(len(ys)))
            if where == "device":
                return NL.device_pair_table(xs, ys, com, com, "exp%d" % k)
            return NL.PairTable(zb.LookupTable(enc(xs), com, "exp%d.x" % k),
                                zb.LookupTable(enc(ys), com, "exp%d.y" % k), "exp%d" % k)

        def rng_table(vals, name):
            com = StubCommitment(_log2(len(vals)))
            if where == "device":
                return NL.device_range_table(vals[0], len(vals), spec, com, name)
            return zb.LookupTable(enc(vals), com, name)

        ts = NL.TableSet(params, 1e-5, p, b"", tuple(pair(k) for k in range(3)), None, None, None,
                         rng_table(t["quant_range"], "quant_range"),
                         rng_table(t["residue_range"], "residue_range"))
        n = _log2(len(c["z"]))
        z_t = _operand(c["z"], 0, n, p, where)
        p_t = _operand(c["p"], 0, n, p, where)
        wit = (c["xi_prime"], c["digits"], c["partials"], [tuple(x) for x in c["chain"]], c["p"])
        tr = Transcript.from_state(bytes.fromhex(c["state_before"]), p)
        pr = zb.prove_softmax_row(z_t, p_t, wit, ts, KEY, tr, _Rng())
        assert list(pr.decomposition_opening.values) == c["decomposition"]
        for got, want in zip(pr.digit_lookups, c["digit_lookups"]):
            _check_lookup(got, want)
        assert [[list(r.evaluations) for r in x.sumcheck.rounds] for x in pr.chain_prod_proofs] \
            == c["chain_prods"]
        for got, want in zip(pr.chain_rescale_proofs, c["chain_rescales"]):
            _check_lookup(got.quant_lookup, want[0])
            _check_lookup(got.resid_lookup, want[1])
        assert list(pr.normalization_opening.values) == c["normalization"]
        assert tr.state.hex() == c["state_end"]


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("dtype", [torch.int16, torch.int32, torch.int64])
@pytest.mark.parametrize("n", [100, (1 << 16) + 3])
def test_lift_signed_ints(field, dtype, n):
    """D.lift (field.py:54-55 from_signed; look-up-table path for n >= 4096)
    equals v mod p for every entry, extremes included."""
    p = FIELDS[field]
    spec = D.spec_for(p)
    info = torch.iinfo(dtype)
    g = torch.Generator().manual_seed(n)
    t = torch.randint(info.min, info.max, (n,), generator=g, dtype=torch.int64).to(dtype)
    edge = [info.min, info.max, 0, 1, -1, 65535 % (info.max + 1), -65536 % info.min if dtype != torch.int16 else -32768]
    t[: len(edge)] = torch.tensor(edge, dtype=torch.int64).to(dtype)
    got = D.download(D.lift(t.cuda(), spec), spec, n)
    assert got == [int(v) % p for v in t.tolist()]


def test_pair_lookup_lazy_secret_miss_and_collision_free_path():
    """prove_pair_lookup bins an in-table pair secret from its integers and
    never builds the 32-byte x + alpha*y column; a query off its table row
    falls back to the hash probe on the combined value and raises
    ElementNotInTable(first index, x + alpha*y) like lookup.py:96-98."""
    c = load_golden("pair_lookup.json")[0]
    p = FIELDS[c["field"]]
    n = len(c["x"])
    nv = (n - 1).bit_length()

    def pt(vals):
        ref = TensorRef("committed", nv // 2, nv - nv // 2, commitment=StubCommitment(nv))
        t = torch.tensor(vals, dtype=torch.int32).cuda().view(1 << (nv // 2), -1)
        return ProverTensor(None, ref, (), device=DeviceMatrix.from_int_tensor(t))

    tx = torch.tensor(c["table_x"], dtype=torch.int32).cuda()
    ty = torch.tensor(c["table_y"], dtype=torch.int32).cuda()
    pair = NL.PairTable(zb.LookupTable(tx, StubCommitment(7), "silu.x"),
                        zb.LookupTable(ty, StubCommitment(7), "silu.y"), "silu")
    y = list(c["y"])
    y[40] += 1  # off its table row (and, with overwhelming probability, off the table)
    y[90] += 3
    tr = Transcript.from_state(bytes.fromhex(c["state_before"]), p)
    with pytest.raises(zb.ElementNotInTable) as e:
        zb.prove_pair_lookup(b"swiglu/act", pt(c["x"]), pt(y), pair, KEY, tr, _Rng())
    assert e.value.index == 40 and 0 <= e.value.value < p


@pytest.mark.parametrize("n,d", [(1 << 16, (1 << 21) + 5), (20000, 100003), (1 << 16, 7)])
def test_range_count16_hot_bins_tails_and_misses(n, d):
    """The vectorised 16-bit-bin histogram (k_range_count16: int16 queries,
    12288 < n <= 2^16): half-word overflow flushes (a bin hit 2^20 times),
    d % 8 tails, misses reported at their first index, and an unaligned
    column taking the fallback kernel -- all against torch.bincount."""
    from paper_2508_21393_b200 import lookup as L

    spec = D.spec_for(FIELDS["big"])
    lo = -(n // 2)
    tab = NL.device_range_table(lo, n, spec, StubCommitment(_log2(n)), "r")
    g = torch.Generator(device="cuda").manual_seed(d)
    x = torch.randint(lo, lo + n, (d,), device="cuda", generator=g, dtype=torch.int64)
    x[: min(d, 1 << 20)] = lo + 1  # one very hot bin: many 0x8000 flushes
    x[3 * d // 4:] = lo + n - 1
    col = x.to(torch.int16)
    for c in (col, torch.cat([col[:1], col])[1:]):  # aligned, then a misaligned view
        counts, index = L.multiplicities_range(D.LiftedColumn(c, spec), tab, c, tab.int_column)
        want = torch.bincount((x - lo).long(), minlength=n)
        got = torch.tensor(D.download(counts.buf, spec, n), dtype=torch.int64)
        assert torch.equal(got, want.cpu())
        assert torch.equal(index[:d].long(), (x - lo).long())
    if n < (1 << 16):
        bad = col.clone()
        bad[d - 1] = lo + n  # in the tail
        bad[d // 2] = lo - 1
        with pytest.raises(zb.ElementNotInTable) as e:
            L.multiplicities_range(D.LiftedColumn(bad, spec), tab, bad, tab.int_column)
        assert e.value.index == min(d // 2, d - 1)


@pytest.mark.parametrize("field", ["big", "test"])
def test_lift_int16_exhaustive(field):
    """Every int16 value (the table-free k_lift16_direct path for Fr255:
    m R1 - q p with a float64 quotient estimate and one correction) lifts to
    v mod p; a ragged length exercises the tail loop."""
    p = FIELDS[field]
    spec = D.spec_for(p)
    t = torch.arange(-32768, 32768, dtype=torch.int64).to(torch.int16)
    t = torch.cat([t, t[:1234]])
    got = D.download(D.lift(t.cuda(), spec), spec, t.numel())
    assert got == [int(v) % p for v in t.tolist()]
