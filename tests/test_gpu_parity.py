"""GPU parity: the CUDA path (through the C-ABI) against the reference goldens
and the CPU oracle, bit-exact.  Run on a B200: pytest -m gpu.
"""

import os
import random

import numpy as np
import pytest

from conftest import FIELDS, P_BIG, P_TEST, load_golden
import inputs
from oracle import fs, logup, multilinear, prime, sc, zkmat
from oracle.stubcommit import StubBackend

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2508_21393_b200 as zb  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402
from paper_2508_21393_b200.commit_stub import StubCommitment, StubKey  # noqa: E402
from paper_2508_21393_b200.gadgets import DeviceMatrix, ProverTensor, TensorRef  # noqa: E402
from paper_2508_21393_b200.transcript import Transcript  # noqa: E402

KEY = StubKey()
ROOT_DIR = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class _Rng:
    def vector(self, n):
        return [0] * n

    def next(self):
        return 0


RNG = _Rng()


def _tr(state_hex, p):
    return Transcript.from_state(bytes.fromhex(state_hex), p)


# --- field / mle -------------------------------------------------------------------


def test_field_mle_golden():
    g = load_golden("field_mle.json")
    for c in g["batch_inverse"]:
        p = FIELDS[c["field"]]
        if "error" in c:
            with pytest.raises(zb.InversionOfZero) as e:
                zb.batch_inverse(c["values"], p)
            assert str(e.value) == c["error"]
        else:
            assert zb.batch_inverse(c["values"], p) == c["inverse"]
    for c in g["eq"]:
        assert zb.eq_table(c["point"], FIELDS[c["field"]]) == c["table"]
    for c in g["fold"]:
        assert zb.fold_table(c["table"], c["r"], FIELDS[c["field"]]) == c["out"]
    for c in g["mle"]:
        assert zb.mle_evaluate(c["table"], c["point"], FIELDS[c["field"]]) == c["value"]


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("n", [1, 2, 255, 2048, 2049, 100000, (1 << 20) + 7])
def test_batch_inverse_sizes(field, n):
    p = FIELDS[field]
    vals = inputs.field_vec(1000 + n, min(n, 4096), p)
    vals = (vals * (n // len(vals) + 1))[:n]
    vals = [v or 1 for v in vals]
    got = zb.batch_inverse(vals, p)
    idx = [0, n // 2, n - 1] + random.Random(n).sample(range(n), min(n, 50))
    for i in idx:
        assert got[i] * vals[i] % p == 1


@pytest.mark.parametrize("field", ["big", "test"])
def test_batch_inverse_zero_reports_first_index(field):
    p = FIELDS[field]
    vals = list(range(1, 5001))
    vals[3333] = 0
    vals[4444] = 0
    with pytest.raises(zb.InversionOfZero, match="at index 3333"):
        zb.batch_inverse(vals, p)
    vals = list(range(1, 100))
    vals[7] = p  # multiple of p but not a literal zero: reference fails at the end
    with pytest.raises(zb.InversionOfZero) as e:
        zb.batch_inverse(vals, p)
    assert str(e.value) == "cannot invert 0"


@pytest.mark.parametrize("field", ["big", "test"])
def test_eq_table_large_two_level(field):
    p = FIELDS[field]
    pt = inputs.field_vec(77, 15, p)
    spec = D.spec_for(p)
    got = D.download(D.eq_table(pt, spec), spec, 1 << 15)
    hi = multilinear.eq_vec(pt[:7], p)
    lo = multilinear.eq_vec(pt[7:], p)
    for i in random.Random(3).sample(range(1 << 15), 200):
        assert got[i] == hi[i >> 8] * lo[i & 255] % p


# --- sumcheck ----------------------------------------------------------------


@pytest.mark.parametrize("native", [True, False])
def test_sumcheck_golden(native, monkeypatch):
    from paper_2508_21393_b200 import sumcheck as S

    monkeypatch.setattr(S, "NATIVE_TRANSCRIPT", native)
    for c in load_golden("sumcheck.json"):
        p = FIELDS[c["field"]]
        t = _tr(c["state_before"], p)
        terms = [zb.Term(co, tuple(f)) for co, f in c["terms"]]
        claim = zb.SumcheckClaim(c["claimed_sum"], c["tables"], terms, c["degree"], p)
        proof, point = zb.prove_sumcheck(claim, t)
        assert [list(r.evaluations) for r in proof.rounds] == c["rounds"], c["note"]
        assert list(proof.final_values) == c["final_values"], c["note"]
        assert isinstance(proof.rounds, list) and isinstance(proof.final_values, tuple)
        assert point == c["point"]
        assert t.state.hex() == c["state_after"]


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("k,degree,n", [(2, 2, 12), (3, 3, 13), (4, 3, 11), (7, 3, 10),
                                        (8, 3, 9), (1, 1, 14)])
def test_sumcheck_random_vs_oracle(field, k, degree, n):
    p = FIELDS[field]
    rnd = random.Random(k * 100 + n)
    tabs = [inputs.field_vec(rnd.randrange(1 << 30), 1 << n, p) for _ in range(k)]
    terms = []
    for _ in range(rnd.randrange(1, 9)):
        nf = rnd.randrange(0, degree + 1)
        terms.append(zb.Term(rnd.randrange(p), tuple(rnd.randrange(k) for _ in range(nf))))
    claimed = rnd.randrange(p)
    t1 = Transcript(b"rand", p, b"s")
    proof, point = zb.prove_sumcheck(zb.SumcheckClaim(claimed, tabs, terms, degree, p), t1)
    t2 = fs.FS(b"rand", p, b"s")
    rounds, finals, opoint = sc.prove(claimed, tabs, [(x.coefficient, x.factors) for x in terms],
                                      degree, t2)
    assert [r.evaluations for r in proof.rounds] == rounds
    assert proof.final_values == finals
    assert point == opoint and t1.state == t2.state


# the recognised round shapes (persistent engine: lane-mode evaluators, the
# grid-kernel -> cluster-kernel handoff at large n, unused tables folded too)
SHAPES = {
    "prod2": (2, [(0, 1)], 3),
    "prod2-deg2": (2, [(1, 0)], 2),
    "prod2-extra-tables": (4, [(3, 1)], 3),
    "prod3": (3, [(0, 1, 2)], 3),
    "sum2prod2": (3, [(0, 1), (0, 2)], 3),
    "generic-mixed": (3, [(0, 1, 2), (1,), ()], 3),
    "logup": (7, [(0, 1, 2), (0, 3), (0, 4, 5), (1,), (6, 4)], 3),
    "logup-permuted": (7, [(3, 6, 0), (3, 2), (3, 5, 1), (6,), (4, 5)], 3),
    "logup-repeated-k4": (4, [(0, 1, 2), (0, 3), (0, 1, 3), (1,), (2, 1)], 3),
}


@pytest.mark.parametrize("field,n", [("test", 16), ("big", 15), ("big", 6), ("test", 1)])
@pytest.mark.parametrize("shape", list(SHAPES))
def test_sumcheck_shapes_vs_oracle(field, n, shape):
    p = FIELDS[field]
    k, factor_sets, degree = SHAPES[shape]
    rnd = random.Random(n * 31 + k)
    tabs = [inputs.field_vec(rnd.randrange(1 << 30), 1 << n, p) for _ in range(k)]
    terms = [zb.Term(rnd.randrange(p), f) for f in factor_sets]
    claimed = rnd.randrange(p)
    t1 = Transcript(b"shape", p, shape.encode())
    proof, point = zb.prove_sumcheck(zb.SumcheckClaim(claimed, tabs, terms, degree, p), t1)
    t2 = fs.FS(b"shape", p, shape.encode())
    rounds, finals, opoint = sc.prove(claimed, tabs, [(x.coefficient, x.factors) for x in terms],
                                      degree, t2)
    assert [r.evaluations for r in proof.rounds] == rounds
    assert proof.final_values == finals
    assert point == opoint and t1.state == t2.state


# --- zkMat ---------------------------------------------------------------------------


def _mm_data(c):
    if c["data"] is not None:
        a, b, cm = (np.asarray(c["data"][k], dtype=np.int64) for k in ("a", "b", "c"))
        d0, d1, d2 = c["dims"]
        return a.reshape(1 << d0, 1 << d1), b.reshape(1 << d1, 1 << d2), cm.reshape(1 << d0, 1 << d2)
    r, k, co = c["shape"]
    return inputs.matmul_case(c["seed"], r, k, co,
                              tamper=tuple(c["tamper"]) if c["tamper"] else None)


def _dev(arr, dtype):
    return DeviceMatrix.from_int_tensor(torch.from_numpy(np.ascontiguousarray(arr)).to(dtype).cuda())


@pytest.fixture(params=["native", "python"])
def mm_driver(request, monkeypatch):
    """zkl_matmul_prove (one C call per claim) and the Python phase driver."""
    from paper_2508_21393_b200 import gadgets as G

    monkeypatch.setattr(G, "NATIVE_DRIVER", request.param == "native")
    return request.param


@pytest.mark.parametrize("mode", ["i64", "i16", "field"])
def test_matmul_sumcheck_golden(mode, mm_driver):
    for c in load_golden("matmul.json"):
        p = FIELDS[c["field"]]
        a, b, cm = _mm_data(c)
        dims = tuple(c["dims"])
        if mode == "field":
            spec = D.spec_for(p)
            A = DeviceMatrix.from_field_list(inputs.to_field(a, p), *a.shape, spec)
            B = DeviceMatrix.from_field_list(inputs.to_field(b, p), *b.shape, spec)
            C = DeviceMatrix.from_field_list(inputs.to_field(cm, p), *cm.shape, spec)
        elif mode == "i16":
            if np.abs(cm).max() >= (1 << 15):
                A, B = _dev(a, torch.int16), _dev(b, torch.int16)
                C = _dev(cm, torch.int64)
            else:
                A, B, C = (_dev(x, torch.int16) for x in (a, b, cm))
        else:
            A, B, C = (_dev(x, torch.int64) for x in (a, b, cm))
        t = _tr(c["state_before"], p)
        rounds, point, finals = zb.matmul_sumcheck(A, B, C, dims, t)
        assert [list(r) for r in rounds] == c["rounds"], (mode, c["shape"])
        assert list(finals) == c["final_values"]
        assert t.state.hex() == c["state_after"]


def test_prove_matmul_full_with_stub_openings(mm_driver):
    """Whole gadget (gadgets.py:230-265) from the pre-absorption state."""
    for c in load_golden("matmul.json"):
        p = FIELDS[c["field"]]
        a, b, cm = _mm_data(c)
        d0, d1, d2 = c["dims"]

        def pt(arr, rv, cv):
            ref = TensorRef("committed", rv, cv, commitment=StubCommitment(rv + cv))
            return ProverTensor(None, ref, (), device=_dev(arr, torch.int64))

        t = _tr(c["state_in"], p)
        proof = zb.prove_matmul(pt(a, d0, d1), pt(b, d1, d2), pt(cm, d0, d2), KEY, t, RNG)
        assert proof.dims == (d0, d1, d2)
        assert [list(r.evaluations) for r in proof.sumcheck.rounds] == c["rounds"]
        assert list(proof.sumcheck.final_values) == c["final_values"]
        assert [list(o.values) for o in (proof.a_opening, proof.b_opening,
                                          proof.c_opening)] == c["openings"]
        assert t.state.hex() == c["state_end"]


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("dims,dt", [((5, 9, 3), "i16"), ((0, 10, 2), "i16"), ((7, 0, 7), "i16"),
                                     ((4, 6, 0), "i64"), ((8, 8, 8), "i16"), ((6, 4, 9), "i32")])
def test_matmul_factored_vs_oracle(field, dims, dt, mm_driver):
    p = FIELDS[field]
    d0, d1, d2 = dims
    g = inputs.rng(sum(dims) * 7 + len(dt))
    a = g.integers(-32768, 32768, size=(1 << d0, 1 << d1))
    b = g.integers(-32768, 32768, size=(1 << d1, 1 << d2))
    cm = a @ b
    cm[0, 0] += 3  # a false claim exercises the non-zero U phase
    tdt = {"i16": torch.int16, "i32": torch.int32, "i64": torch.int64}[dt]
    A, B = _dev(a, tdt), _dev(b, tdt)
    C = _dev(cm, torch.int64)
    t1 = Transcript(b"mm", p, b"x")
    rounds, point, finals = zb.matmul_sumcheck(A, B, C, dims, t1)
    t2 = fs.FS(b"mm", p, b"x")
    orounds, ofinals, opoint = zkmat.prove_factored(a.reshape(-1), b.reshape(-1), cm.reshape(-1),
                                                    dims, t2)
    assert rounds == orounds and tuple(finals) == ofinals and point == opoint
    assert t1.state == t2.state


@pytest.mark.parametrize("field", ["big", "test"])
def test_matmul_batch_matches_per_claim(field):
    """matmul_sumcheck_batch (one native call, the next claim's draws and
    matvecs queued behind the previous claim's last fold) against the
    per-claim loop with the same transcript records: identical rounds,
    points, finals, end state and transcript log; claims with empty
    dimensions (d0 = 0, d1 = 0, d2 = 0), a false claim, and mixed integer
    types, each checked against the oracle as well."""
    p = FIELDS[field]
    g = inputs.rng(31 + len(field))
    specs = [((5, 9, 3), torch.int16), ((0, 10, 2), torch.int16), ((4, 6, 0), torch.int64),
             ((8, 8, 8), torch.int16), ((7, 0, 7), torch.int32), ((6, 4, 9), torch.int16)]
    claims, host = [], []
    for i, (dims, tdt) in enumerate(specs):
        d0, d1, d2 = dims
        a = g.integers(-32768, 32768, size=(1 << d0, 1 << d1))
        b = g.integers(-32768, 32768, size=(1 << d1, 1 << d2))
        cm = a @ b
        if i == 3:
            cm[1, 2] -= 5  # a false claim
        claims.append((_dev(a, tdt), _dev(b, tdt), _dev(cm, torch.int64), dims))
        host.append((a, b, cm, dims))
    pre = [[(b"gadget/tag", b"matmul"), (b"claim", b"%d" % i), (b"n", i * 1000 + 7)]
           for i in range(len(claims))]
    t1 = Transcript(b"batch", p, b"s")
    got = zb.matmul_sumcheck_batch(claims, t1, pre)
    t2 = Transcript(b"batch", p, b"s")
    want = []
    for c, recs in zip(claims, pre):
        for label, data in recs:
            t2.append(label, data)
        want.append(zb.matmul_sumcheck(*c, t2))
    assert got == want
    assert t1.state == t2.state and t1.log == t2.log
    t3 = fs.FS(b"batch", p, b"s")
    for (a, b, cm, dims), recs, (rounds, point, finals) in zip(host, pre, got):
        for label, data in recs:
            t3.append(label, data)
        orounds, ofinals, opoint = zkmat.prove_factored(a.reshape(-1), b.reshape(-1),
                                                        cm.reshape(-1), dims, t3)
        assert rounds == orounds and tuple(finals) == ofinals and point == opoint
    assert t3.state == t1.state


def _run_isolated(code, **env):
    import subprocess
    import sys

    return subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                          cwd=ROOT_DIR, env=dict(os.environ, **env))


def test_graph_cache_survives_arena_growth():
    """The zkMat phase inputs replay from a CUDA-graph cache keyed by the
    operand and workspace pointers and the arenas' generation: prove a claim
    until its graphs are captured and replayed, grow the work arena underneath
    (a claim with much longer vectors), and prove again -- every proof equals
    the oracle's."""
    p = P_BIG
    dims = (7, 8, 6)
    g = inputs.rng(77)
    a = g.integers(-32768, 32768, size=(1 << dims[0], 1 << dims[1]))
    b = g.integers(-32768, 32768, size=(1 << dims[1], 1 << dims[2]))
    cm = a @ b
    A, B, C = _dev(a, torch.int16), _dev(b, torch.int16), _dev(cm, torch.int64)
    t2 = fs.FS(b"gc", p, b"x")
    want = zkmat.prove_factored(a.reshape(-1), b.reshape(-1), cm.reshape(-1), dims, t2)
    for it in range(5):
        if it == 3:  # grow the work arena: a claim with 2^14-entry vectors
            bd = (14, 4, 6)
            ba = g.integers(-9, 9, size=(1 << bd[0], 1 << bd[1]))
            bb = g.integers(-9, 9, size=(1 << bd[1], 1 << bd[2]))
            zb.matmul_sumcheck(_dev(ba, torch.int16), _dev(bb, torch.int16),
                               _dev(ba @ bb, torch.int64), bd, Transcript(b"big", p, b"y"))
        t1 = Transcript(b"gc", p, b"x")
        rounds, point, finals = zb.matmul_sumcheck(A, B, C, dims, t1)
        assert rounds == want[0] and tuple(finals) == want[1] and point == want[2], it
        assert t1.state == t2.state


def test_zero_u_phase_shortcut_off_matches_golden():
    """A true claim's U phase is proven on the host (h = A B E_v - C E_v is
    identically zero, so every round polynomial is zero); with the shortcut
    off (ZKL_NO_ZERO_PHASE=1) the device rounds give the same bytes: both
    are checked against the reference's goldens and the batch test."""
    code = (
        "import sys; sys.path[:0] = ['.', 'tests', 'tests/golden']\n"
        "import test_gpu_parity as T\n"
        "for mode in ('i16', 'i64', 'field'):\n"
        "    T.test_matmul_sumcheck_golden(mode, 'native')\n"
        "T.test_matmul_batch_matches_per_claim('big')\n"
        "T.test_matmul_batch_matches_per_claim('test')\n"
        "print('ok')\n")
    r = _run_isolated(code, ZKL_NO_ZERO_PHASE="1")
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


@pytest.mark.parametrize("tail,paired", [("0", "1"), ("1", "1"), ("6", "1"), ("5", "0"),
                                         ("5", "64"), ("3", "64")])
def test_host_tail_rounds_match_golden(tail, paired):
    """The last ZKL_HOST_TAIL rounds of a phase run on the host (default 5;
    the cluster kernel sends the folded survivors through the mailbox).  With
    every round on the device (0), one host round (1) and six (6), the
    sumcheck and zkMat proofs are the reference's goldens, constant terms,
    repeated factors and post_add rounds included.  `paired`: the cluster
    kernel's paired rounds (PROD2 / SUM2PROD2, one round trip per two rounds)
    on by default ("1"), off ("0"), or from round 0 on (ZKL_PAIR_PASSES=64:
    multi-pass pair passes, the unfolded first pass and the double folds)."""
    code = (
        "import sys; sys.path[:0] = ['.', 'tests', 'tests/golden']\n"
        "import pytest, test_gpu_parity as T\n"
        "mp = pytest.MonkeyPatch()\n"
        "T.test_sumcheck_golden(True, mp)\n"
        "for mode in ('i16', 'i64', 'field'):\n"
        "    T.test_matmul_sumcheck_golden(mode, 'native')\n"
        "T.test_matmul_batch_matches_per_claim('big')\n"
        "print('ok')\n")
    env = {"ZKL_HOST_TAIL": tail}
    if paired == "0":
        env["ZKL_PAIRED"] = "0"
    elif paired != "1":
        env["ZKL_PAIR_PASSES"] = paired
    r = _run_isolated(code, **env)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


def test_stepwise_mode_matches_oracle():
    """ZKL_NO_PERSISTENT=1 (what profilers get automatically): one launch per
    round through the same drivers, still bit-exact."""
    code = (
        "import sys; sys.path[:0] = ['.', 'tests', 'tests/golden']\n"
        "import test_gpu_parity as T\n"
        "class M: pass\n"
        "T.test_matmul_factored_vs_oracle('big', (5, 9, 3), 'i16', 'native')\n"
        "T.test_matmul_factored_vs_oracle('test', (0, 10, 2), 'i16', 'native')\n"
        "T.test_matmul_factored_vs_oracle('big', (7, 0, 7), 'i16', 'native')\n"
        "T.test_sumcheck_shapes_vs_oracle('big', 6, 'sum2prod2')\n"
        "T.test_sumcheck_shapes_vs_oracle('test', 16, 'prod3')\n"
        "print('ok')\n")
    r = _run_isolated(code, ZKL_NO_PERSISTENT="1")
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


def test_profile_replay_mode_matches_oracle():
    """ZKL_PROFILE_REPLAY=1 (the ncu capture mode for the production
    kernels): each phase is proven stepwise, then re-run by the persistent /
    cluster kernels on recorded challenges, whose final folded values must
    equal the proof's (the driver raises otherwise).  Proofs stay bit-exact,
    including a dense claim large enough for the grid -> cluster handoff."""
    code = (
        "import sys; sys.path[:0] = ['.', 'tests', 'tests/golden']\n"
        "import test_gpu_parity as T\n"
        "T.test_sumcheck_shapes_vs_oracle('big', 6, 'sum2prod2')\n"
        "T.test_sumcheck_shapes_vs_oracle('test', 16, 'prod3')\n"
        "T.test_sumcheck_random_vs_oracle('big', 7, 3, 12)\n"
        "T.test_matmul_factored_vs_oracle('big', (5, 9, 3), 'i16', 'native')\n"
        "import test_gpu_parity_scale as S\n"
        "S.test_cfg5_dense_replicated_claim_matches_oracle()\n"
        "print('ok')\n")
    r = _run_isolated(code, ZKL_PROFILE_REPLAY="1")
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


@pytest.mark.parametrize("env", [{"ZKL_MATVEC_SLOW": "1"},
                                 {"ZKL_MV_TC64": "0", "ZKL_MATVEC_FAST64": "1"},
                                 {"ZKL_MV_TC64": "0"}, {"ZKL_MV_TC": "0"}])
def test_matvec_alternate_kernels_vs_numpy(env):
    """The non-default matvec kernels (wide-accumulator everywhere; int64 on
    mad.wide or on the wide-accumulator kernels instead of the tensor cores;
    int16 on mad.wide; the switches are read once per process) against exact
    numpy products, in a child process."""
    code = (
        "import sys; sys.path[:0] = ['.', 'tests', 'tests/golden']\n"
        "import test_gpu_parity as T\n"
        "for mt in ('i16', 'i64'):\n"
        "    for shape in [(64, 256), (1024, 256), (33, 4096), (256, 1024), (3, 70)]:\n"
        "        T.test_matvec_extremes_vs_numpy('big', mt, shape)\n"
        "print('ok')\n")
    r = _run_isolated(code, **env)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("mt", ["i16", "i32", "i64"])
@pytest.mark.parametrize("shape", [(1, 1), (3, 70), (64, 5), (1024, 256), (33, 4096),
                                   (40, 1030)])
def test_matvec_extremes_vs_numpy(field, mt, shape):
    from paper_2508_21393_b200.gadgets import _matvec

    p = FIELDS[field]
    spec = D.spec_for(p)
    lo, hi = {"i16": (-32768, 32767), "i32": (-2**31, 2**31 - 1), "i64": (-2**63, 2**63 - 1)}[mt]
    g = inputs.rng(shape[0] * 31 + shape[1])
    M = g.integers(lo, hi, size=shape, dtype=np.int64, endpoint=True)
    M.flat[0] = lo
    M.flat[-1] = hi
    tdt = {"i16": torch.int16, "i32": torch.int32, "i64": torch.int64}[mt]
    Md = _dev(M, tdt)
    for transpose in (0, 1):
        xlen = shape[0] if transpose else shape[1]
        x = inputs.field_vec(xlen + transpose, xlen, p)
        y = D.download(_matvec(Md, D.upload(x, spec), bool(transpose), spec), spec,
                       shape[1] if transpose else shape[0])
        ML = M.T if transpose else M
        want = [sum(int(v) * x[j] for j, v in enumerate(row)) % p for row in ML.tolist()]
        assert y == want, transpose


def test_elementprod_golden():
    for c in load_golden("elementprod.json"):
        p = FIELDS[c["field"]]
        rv, cv = ((x - 1).bit_length() for x in c["shape"])

        def pt(vals):
            ref = TensorRef("committed", rv, cv, commitment=StubCommitment(rv + cv))
            arr = np.asarray(vals, dtype=np.int64).reshape(1 << rv, 1 << cv)
            return ProverTensor(None, ref, (), device=_dev(arr, torch.int64))

        t = _tr(c["state_in"], p)
        proof = zb.prove_elementprod(pt(c["a"]), pt(c["b"]), pt(c["c"]), KEY, t, RNG)
        assert proof.c_opening.values[0] == c["claimed_sum"]
        assert [list(r.evaluations) for r in proof.sumcheck.rounds] == c["rounds"]
        assert list(proof.sumcheck.final_values) == c["final_values"]
        assert list(proof.ab_opening.values) == c["ab_opening"]
        assert t.state.hex() == c["state_end"]


# --- logUp -----------------------------------------------------------------------------


class _PairTable:
    def __init__(self, x, y, name):
        self.x, self.y, self.name = x, y, name


def test_pair_lookup_golden_device():
    """SiLU pair lookup (gadgets.py:679-688) entirely on the GPU: device int
    columns -> x + alpha*y compression -> multiplicities -> logUp; bit-exact
    with the reference's own run (tests/golden/pair_lookup.json)."""
    for c in load_golden("pair_lookup.json"):
        p = FIELDS[c["field"]]
        n = len(c["x"])
        nv = (n - 1).bit_length()

        def pt(vals):
            ref = TensorRef("committed", nv // 2, nv - nv // 2, commitment=StubCommitment(nv))
            t = torch.tensor(vals, dtype=torch.int32).cuda().view(1 << (nv // 2), -1)
            return ProverTensor(None, ref, (), device=DeviceMatrix.from_int_tensor(t))

        tx = torch.tensor(c["table_x"], dtype=torch.int32).cuda()
        ty = torch.tensor(c["table_y"], dtype=torch.int32).cuda()
        pair = _PairTable(zb.LookupTable(tx, StubCommitment(7)), zb.LookupTable(ty, StubCommitment(7)),
                          "silu")
        t = _tr(c["state_before"], p)
        pr = zb.prove_pair_lookup(b"swiglu/act", pt(c["x"]), pt(c["y"]), pair, KEY, t, RNG)
        assert pr.beta_retries == c["beta_retries"]
        assert [list(r.evaluations) for r in pr.sumcheck.rounds] == c["rounds"]
        assert list(pr.sumcheck.final_values) == c["final_values"]
        assert list(pr.secret_values) == c["secret_values"]
        assert list(pr.table_values) == c["table_values"]
        assert t.state.hex() == c["state_end"]


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("n", [1000, (1 << 18) + 3])
def test_pair_combine_vs_python(field, n):
    """x + alpha*y over signed int16 columns (gadgets.py:659-666): the
    lookup-table path (n >= 2^18) and the direct path, incl. -32768/32767."""
    p = FIELDS[field]
    spec = D.spec_for(p)
    g = inputs.rng(n)
    x = g.integers(-32768, 32768, size=n).astype(np.int16)
    y = g.integers(-32768, 32768, size=n).astype(np.int16)
    x[:2] = (-32768, 32767)
    y[:2] = (32767, -32768)
    alpha = (p - 12345) * 3 % p
    dv = D.pair_combine(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), alpha, spec)
    m = min(n, 4096)
    got = D.download(dv.buf, spec, m)
    want = [(int(a) + alpha * int(b)) % p for a, b in zip(x[:m], y[:m])]
    assert got == want
    tail = D.download(dv.buf, spec, n)[-100:]
    assert tail == [(int(a) + alpha * int(b)) % p for a, b in zip(x[-100:], y[-100:])]


def test_multiplicities_skewed_warp_aggregation():
    """Heavily repeated secrets (the zero padding of a lookup) through the
    warp-aggregated histogram."""
    p = P_TEST
    table = list(range(1000, 1000 + 4096))
    secret = [1000] * 5000 + [1000 + (i * 7) % 4096 for i in range(3000)] + [5095] * 192
    tab = zb.LookupTable(tuple(table), None)
    got = zb.compute_multiplicities(secret, tab, p)
    assert got == logup.multiplicities(secret, table)


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("d,n", [(1 << 18, 1 << 12), (1 << 12, 1 << 2), (1 << 16, 1 << 15)])
def test_lookup_tiled_matches_materialised(field, d, n, monkeypatch):
    """The tiled logUp path (replicated table side never materialised) and the
    fully materialised 7-table claim give identical proofs."""
    from paper_2508_21393_b200 import lookup as L

    p = FIELDS[field]
    spec = D.spec_for(p)
    rnd = np.random.default_rng(d + n)
    table = [int(v) for v in rnd.integers(0, 2**40, size=n)]
    idx = rnd.integers(0, n, size=d)
    sec = D.upload([table[int(i)] for i in idx], spec)
    tab = zb.LookupTable(D.DeviceVector(D.upload(table, spec), n, spec), StubCommitment(
        (n - 1).bit_length()))
    secret = zb.SecretVector(D.DeviceVector(sec, d, spec), StubCommitment((d - 1).bit_length()), ())
    out = []
    for tiled in (True, False):
        monkeypatch.setattr(L, "TILED", tiled)
        m = zb.compute_multiplicities(secret.entries, tab)
        t = Transcript(b"tiled", p, b"x")
        pr = zb.prove_lookup(secret, m, tab, KEY, t, RNG)
        out.append(([r.evaluations for r in pr.sumcheck.rounds], pr.sumcheck.final_values,
                     pr.secret_values, pr.table_values, t.state))
    assert out[0] == out[1]


def _indexed_lookup_proofs(p, table, secret_vals, monkeypatch, label=b"x"):
    """One proof per (tiled, indexed) combination over device-resident entries."""
    from paper_2508_21393_b200 import lookup as L

    spec = D.spec_for(p)
    d, n = len(secret_vals), len(table)
    tab = zb.LookupTable(D.DeviceVector(D.upload(table, spec), n, spec), StubCommitment(
        (n - 1).bit_length()))
    secret = zb.SecretVector(D.DeviceVector(D.upload(secret_vals, spec), d, spec),
                             StubCommitment((d - 1).bit_length()), ())
    out = []
    for tiled in (True, False):
        for indexed in (False, True):
            monkeypatch.setattr(L, "TILED", tiled)
            t = Transcript(b"tiled", p, label)
            if indexed:
                m, index = L.multiplicities_indexed(secret.entries, tab)
                pr = zb.prove_lookup(secret, m, tab, KEY, t, RNG, secret_index=index)
            else:
                m = zb.compute_multiplicities(secret.entries, tab)
                pr = zb.prove_lookup(secret, m, tab, KEY, t, RNG)
            out.append((pr.beta_retries, [r.evaluations for r in pr.sumcheck.rounds],
                        pr.sumcheck.final_values, pr.secret_values, pr.table_values, t.state))
    return out


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("d,n", [(1 << 16, 1 << 10), (1 << 8, 1 << 12), (1 << 12, 1 << 12)])
def test_lookup_indexed_matches_plain(field, d, n, monkeypatch):
    """Secret-side columns gathered through the multiplicity index (no
    d-entry inversion) give the same proofs as inverting the secret, on the
    tiled and the materialised path; the table holds duplicate values (the
    index points at the last one, lookup.py:94)."""
    p = FIELDS[field]
    rnd = np.random.default_rng(d * 3 + n)
    table = [int(v) for v in rnd.integers(0, 2**40, size=n)]
    table[1] = table[n - 1]
    table[2] = table[n // 2]
    sec = [table[int(i)] for i in rnd.integers(0, n, size=d)]
    sec[0] = table[1]
    out = _indexed_lookup_proofs(p, table, sec, monkeypatch)
    assert all(o == out[0] for o in out[1:])


def test_lookup_indexed_pole_retry(monkeypatch):
    """beta landing on a pole (beta + t_j == 0, with t_j also a secret entry):
    the indexed path retries exactly like the plain one (lookup.py:163-171)."""
    p = P_BIG
    rnd = np.random.default_rng(77)
    n, d = 1 << 8, 1 << 12
    table = [int(v) for v in rnd.integers(0, 2**40, size=n)]
    sec = [table[int(i)] for i in rnd.integers(0, n, size=d)]

    betas = []

    class _Capture(Transcript):
        def challenge(self, label):
            v = super().challenge(label)
            if label == b"lookup/beta":
                betas.append(v)
            return v

    spec = D.spec_for(p)
    tab = zb.LookupTable(D.DeviceVector(D.upload(table, spec), n, spec), StubCommitment(8))
    secret = zb.SecretVector(D.DeviceVector(D.upload(sec, spec), d, spec), StubCommitment(12), ())
    t = _Capture(b"tiled", p, b"pole")
    zb.prove_lookup(secret, zb.compute_multiplicities(secret.entries, tab), tab, KEY, t, RNG)
    pole = (p - betas[0]) % p  # the stub commitments do not depend on the entries
    old = table[5]
    table[5] = pole
    sec = [table[6] if v == old else v for v in sec]
    sec[100] = pole
    out = _indexed_lookup_proofs(p, table, sec, monkeypatch, label=b"pole")
    assert out[0][0] >= 1
    assert all(o == out[0] for o in out[1:])


@pytest.mark.parametrize("xdt", [torch.int16, torch.int32])
def test_pair_multiplicities_direct(xdt):
    """Direct binning of pair queries (table x column = consecutive range) gives
    the same counts, indices and first miss as hashing the combined values,
    including queries whose y disagrees with the table (hash fallback)."""
    from paper_2508_21393_b200 import lookup as L

    p = P_BIG
    spec = D.spec_for(p)
    rnd = np.random.default_rng(5)
    n, d, x0 = 4096, 1 << 16, -2048
    tx = torch.arange(x0, x0 + n, dtype=torch.int32).cuda()
    ty = torch.from_numpy(rnd.integers(-30000, 30000, size=n).astype(np.int32)).cuda()
    idx = rnd.integers(0, n, size=d)
    xq = torch.from_numpy((idx + x0).astype(np.int64)).to(xdt).cuda()
    yq = ty.cpu()[torch.from_numpy(idx)].to(xdt).cuda()
    alpha = 987654321987654321
    tab = zb.LookupTable(D.pair_combine(tx, ty, alpha, spec), None)
    sec = D.pair_combine(xq, yq, alpha, spec)
    got = L.multiplicities_pair(sec, tab, xq, yq, tx, ty)
    assert got is not None
    want = L.multiplicities_indexed(sec, tab)
    assert D.as_list(got[0]) == D.as_list(want[0])
    assert torch.equal(got[1][:d], want[1][:d])
    # a query whose (x, y) is not a table pair but whose combined value is a
    # table value takes the hash fallback and still lands in its bin
    xq3 = xq.clone()
    xq3[9] = x0 + n + 5
    got3 = L.multiplicities_pair(sec, tab, xq3, yq, tx, ty)
    assert D.as_list(got3[0]) == D.as_list(want[0])
    assert torch.equal(got3[1][:d], want[1][:d])
    yq2 = yq.clone()
    yq2[7] = yq2[7] + 1  # now (x, y) is not a table pair: combined value misses
    sec2 = D.pair_combine(xq, yq2, alpha, spec)
    with pytest.raises(zb.ElementNotInTable) as e1:
        L.multiplicities_pair(sec2, tab, xq, yq2, tx, ty)
    with pytest.raises(zb.ElementNotInTable) as e2:
        L.multiplicities_indexed(sec2, tab)
    assert e1.value.index == e2.value.index == 7


def test_pair_multiplicities_duplicate_table_declines():
    """A combined table with a repeated value (the reference maps it to the
    last index) is left to the hash path."""
    from paper_2508_21393_b200 import lookup as L

    p = P_TEST
    spec = D.spec_for(p)
    n = 64
    tx = torch.arange(0, n, dtype=torch.int32).cuda()
    ty = torch.zeros(n, dtype=torch.int32).cuda()
    vals = list(range(n))
    vals[10] = vals[20]  # duplicate combined value
    tab = zb.LookupTable(D.DeviceVector(D.upload(vals, spec), n, spec), None)
    xq = torch.tensor([3, 20, 10], dtype=torch.int16).cuda()
    yq = torch.zeros(3, dtype=torch.int16).cuda()
    sec = D.DeviceVector(D.upload([3, 20, 20], spec), 3, spec)
    assert L.multiplicities_pair(sec, tab, xq, yq, tx, ty) is None
    counts, index = L.multiplicities_indexed(sec, tab)
    assert D.as_list(counts)[20] == 2 and D.as_list(counts)[10] == 0


@pytest.mark.parametrize("indexed", [False, True])
def test_lookup_pole_collision_after_max_retries(indexed):
    """beta hitting a pole four times in a row raises PoleCollision
    (lookup.py:165-171: three retries, each absorbing b"lookup/beta-retry"),
    like the oracle; three poles still prove with beta_retries == 3."""
    from oracle.stubcommit import stub_bytes
    from paper_2508_21393_b200 import lookup as L

    p = P_BIG
    spec = D.spec_for(p)
    rnd = np.random.default_rng(91)
    n, d = 1 << 8, 1 << 10
    base = [int(v) for v in rnd.integers(0, 2**40, size=n)]
    betas = []

    class _Capture(Transcript):
        def challenge(self, label):
            v = super().challenge(label)
            if label == b"lookup/beta":
                betas.append(v)
            return v

    def run(table, tr_cls=Transcript):
        tab = zb.LookupTable(D.DeviceVector(D.upload(table, spec), n, spec), StubCommitment(8))
        sec = zb.SecretVector(D.DeviceVector(D.upload([table[10]] * d, spec), d, spec),
                              StubCommitment(10), ())
        t = tr_cls(b"pole", p, b"x")
        if indexed:
            m, index = L.multiplicities_indexed(sec.entries, tab)
            return zb.prove_lookup(sec, m, tab, KEY, t, RNG, secret_index=index)
        return zb.prove_lookup(sec, zb.compute_multiplicities(sec.entries, tab), tab, KEY, t, RNG)

    table = list(base)
    for k in range(4):  # place -beta_k at position k: the next run retries once more
        betas.clear()
        pr = run(table, _Capture)
        assert pr.beta_retries == k
        table[k] = (p - betas[-1]) % p
        if k == 3:
            break
    with pytest.raises(zb.PoleCollision):
        run(table)
    with pytest.raises(logup.Pole):
        mult = logup.multiplicities([table[10]] * d, table)
        logup.prove([table[10]] * d, mult, table, stub_bytes(8), stub_bytes(10),
                    fs.FS(b"pole", p, b"x"), StubBackend(p))


def test_multiplicities_golden():
    for c in load_golden("lookup.json")["multiplicities"]:
        table = zb.LookupTable(tuple(c["table"]), None)
        if "error" in c:
            with pytest.raises(zb.ElementNotInTable) as e:
                zb.compute_multiplicities(c["secret"], table)
            assert [e.value.index, e.value.value] == c["error"]
        else:
            assert zb.compute_multiplicities(c["secret"], table) == c["counts"]


def test_multiplicities_large_vs_oracle():
    rnd = random.Random(8)
    table = [rnd.randrange(P_BIG) for _ in range(1 << 12)]
    table[5] = table[900]  # duplicate: last index wins
    secret = [rnd.choice(table) for _ in range(1 << 16)]
    got = zb.compute_multiplicities(secret, zb.LookupTable(tuple(table), None))
    assert got == logup.multiplicities(secret, table)
    secret[40000] = 12345
    secret[50000] = 54321
    with pytest.raises(zb.ElementNotInTable) as e:
        zb.compute_multiplicities(secret, zb.LookupTable(tuple(table), None))
    assert e.value.index == 40000


def _lookup_run(c):
    p = FIELDS[c["field"]]
    d, n = len(c["secret"]), len(c["table"])
    table = zb.LookupTable(tuple(c["table"]), StubCommitment((n - 1).bit_length()))
    secret = zb.SecretVector(tuple(c["secret"]), StubCommitment((d - 1).bit_length()), ())
    t = _tr(c["state_before"], p)
    return zb.prove_lookup(secret, list(c["mult"]), table, KEY, t, RNG), t


def test_lookup_golden():
    for c in load_golden("lookup.json")["lookup"]:
        proof, t = _lookup_run(c)
        assert proof.beta_retries == c["beta_retries"]
        assert [list(r.evaluations) for r in proof.sumcheck.rounds] == c["rounds"], c["note"]
        assert list(proof.sumcheck.final_values) == c["final_values"], c["note"]
        assert list(proof.secret_values) == c["secret_values"], c["note"]
        assert list(proof.table_values) == c["table_values"], c["note"]
        assert t.state.hex() == c["state_end"], c["note"]


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("d,n", [(1 << 14, 1 << 10), (1 << 8, 1 << 12), (1 << 10, 1 << 10)])
def test_lookup_vs_oracle(field, d, n):
    p = FIELDS[field]
    rnd = random.Random(d + n)
    table = [rnd.randrange(p) for _ in range(n)]
    secret = [rnd.choice(table) for _ in range(d)]
    mult = logup.multiplicities(secret, table)
    nb = lambda k: (k - 1).bit_length()  # noqa: E731
    t1 = Transcript(b"lk", p, b"q")
    proof = zb.prove_lookup(zb.SecretVector(tuple(secret), StubCommitment(nb(d)), ()), mult,
                            zb.LookupTable(tuple(table), StubCommitment(nb(n))), KEY, t1, RNG)
    t2 = fs.FS(b"lk", p, b"q")
    from oracle.stubcommit import stub_bytes

    out = logup.prove(secret, mult, table, stub_bytes(nb(n)), stub_bytes(nb(d)), t2,
                      StubBackend(p))
    assert [r.evaluations for r in proof.sumcheck.rounds] == out["rounds"]
    assert proof.sumcheck.final_values == out["final_values"]
    assert proof.secret_values == out["secret_values"]
    assert proof.table_values == out["table_values"]
    assert t1.state == t2.state


def test_cfg2_xw_full_size_matches_oracle():
    """BASELINE cfg2's largest claim, Y1 = X.W at LLaMA-2-7B shape (11,12,12:
    the reference's replicated form would be 4 x 2^35 entries), proven on the
    GPU and by the oracle's factored restatement (validated bit-exact against
    the reference on small shapes): identical rounds, finals, end state."""
    import bench

    name, a, b, c, dims = [cl for cl in bench.cfg2_claims(1234, "cuda") if cl[0] == "Y1=X.W"][0]
    assert dims == (11, 12, 12)
    tr1 = zb.Transcript(b"check", P_BIG, b"x")
    r1 = zb.matmul_sumcheck(DeviceMatrix.from_int_tensor(a), DeviceMatrix.from_int_tensor(b),
                            DeviceMatrix.from_int_tensor(c), dims, tr1)
    tr2 = fs.FS(b"check", P_BIG, b"x")
    r2 = zkmat.prove_factored(a.cpu().numpy().astype(np.int64).reshape(-1),
                              b.cpu().numpy().astype(np.int64).reshape(-1),
                              c.cpu().numpy().reshape(-1), dims, tr2)
    assert r1[0] == r2[0] and tuple(r1[2]) == r2[1] and tr1.state == tr2.state
