"""Sharded proving (paper_2508_21393_b200/shard.py + csrc/shard.cu) on the GPU:
G rank processes, each proving its cyclic low-bit shard of the same claim
through the native sharded engine, must each return exactly the unsharded
prover's rounds, point, finals and end transcript state.

Every run here gets one GPU, so the G ranks share cuda:0 and run the
engine's stepwise mode (ZKL_NO_PERSISTENT=1: a round is one short fold +
evaluation launch on the rank's own shard, and the ranks wait for each other
on the host, never inside a kernel).  On a multi-GPU node each rank runs the
persistent engine on its own device with the exchange inside the host round
loop; that path is exercised here with a one-rank group (the exchange is then
with itself), bit-exact against the unsharded prover."""

import random
import secrets

import pytest

from conftest import FIELDS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.multiprocessing as mp  # noqa: E402


def _claim(field, n, seed):
    import inputs

    p = FIELDS[field]
    rnd = random.Random(seed)
    tabs = [inputs.field_vec(rnd.randrange(1 << 30), 1 << n, p) for _ in range(3)]
    terms = [(rnd.randrange(p), (0, 1, 2)), (rnd.randrange(p), (1,)), (rnd.randrange(p), (0, 2))]
    post_add = [rnd.randrange(p) for _ in range(n)]
    post_mul = rnd.randrange(p)
    return p, tabs, terms, post_add, post_mul


def _stepwise():
    import os

    os.environ["ZKL_NO_PERSISTENT"] = "1"  # ranks share this test box's one GPU


def _generic_worker(rank, world, name, field, n, seed, q):
    import sys

    _stepwise()
    sys.path[:0] = [".", "tests", "tests/golden"]
    import paper_2508_21393_b200 as zb
    from paper_2508_21393_b200 import device as D
    from paper_2508_21393_b200 import shard

    torch.cuda.set_device(0)
    p, tabs, terms, post_add, post_mul = _claim(field, n, seed)
    spec = D.spec_for(p)
    with shard.ShardGroup(name, rank, world):
        loc = [D.upload(t[rank::world], spec) for t in tabs]
        tr = zb.Transcript(b"shard", p, b"seed")
        zb.sumcheck.absorb_claim(tr, 0, [zb.Term(c, f) for c, f in terms], 3, n)
        out = shard.run_rounds_sharded(spec, loc, n, terms, 3, tr, post_add=post_add,
                                       post_mul=post_mul)
        q.put((rank, out, bytes(tr.state)))


def _spawn(target, world, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = "g" + secrets.token_hex(6)
    ps = [ctx.Process(target=target, args=(r, world, name) + args + (q,)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=600) for _ in ps))
    for p in ps:
        p.join(timeout=120)
    return res


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("field,n", [("big", 12), ("test", 14)])
def test_sharded_generic_claim_matches_unsharded(field, n, world):
    import paper_2508_21393_b200 as zb
    from paper_2508_21393_b200 import device as D
    from paper_2508_21393_b200.sumcheck import run_rounds

    res = _spawn(_generic_worker, world, (field, n, 5 * n + world))
    p, tabs, terms, post_add, post_mul = _claim(field, n, 5 * n + world)
    spec = D.spec_for(p)
    tr = zb.Transcript(b"shard", p, b"seed")
    zb.sumcheck.absorb_claim(tr, 0, [zb.Term(c, f) for c, f in terms], 3, n)
    want = run_rounds(spec, [D.upload(t, spec) for t in tabs], n, terms, 3, tr,
                      post_add=post_add, post_mul=post_mul)
    for r in range(world):
        (rounds, point, finals), state = res[r]
        assert rounds == want[0] and point == want[1] and finals == want[2], r
        assert state == bytes(tr.state)


def _gadget_worker(rank, world, name, kind, n, q):
    import sys

    _stepwise()
    sys.path[:0] = [".", "tests", "tests/golden"]
    import paper_2508_21393_b200 as zb
    from paper_2508_21393_b200 import shard

    torch.cuda.set_device(0)
    with shard.ShardGroup(name, rank, world):
        q.put((rank,) + _gadget(kind, n, zb))


class _Rng:
    def vector(self, k):
        return [0] * k


def _gadget(kind, n, zb):
    """One gadget-level claim; returns (rounds, finals, end state)."""
    from paper_2508_21393_b200.commit_stub import StubCommitment, StubKey
    from paper_2508_21393_b200.gadgets import DeviceMatrix, ProverTensor, TensorRef

    p = FIELDS["big"]
    g = torch.Generator().manual_seed(n)
    tr = zb.Transcript(b"shard-gadget", p, kind.encode())
    if kind == "range_lookup":
        # a rescale-style quant_range lookup: 2^n int16 queries vs the 2^16 table
        from paper_2508_21393_b200 import device as D
        from paper_2508_21393_b200 import nonlinear as NL

        spec = D.spec_for(p)
        tab = NL.device_range_table(-32768, 1 << 16, spec, StubCommitment(16), "quant_range")
        x = torch.randint(-2 ** 15, 2 ** 15, (1 << (n // 2), 1 << (n - n // 2)),
                          generator=g).to(torch.int16).cuda()
        rv, cv = n // 2, n - n // 2
        ref = TensorRef("committed", rv, cv, commitment=StubCommitment(n))
        lp = NL._range_lookup(ProverTensor(None, ref, (), device=DeviceMatrix.from_int_tensor(x)),
                              tab, StubKey(), tr, _Rng())
        return ([tuple(r.evaluations) for r in lp.sumcheck.rounds],
                tuple(lp.sumcheck.final_values) + tuple(lp.secret_values) + tuple(lp.table_values),
                bytes(tr.state))
    if kind == "elementprod":
        rows, cols = 1 << (n // 2), 1 << (n - n // 2)
        a = torch.randint(-2 ** 15, 2 ** 15, (rows, cols), generator=g).to(torch.int16)
        b = torch.randint(-2 ** 15, 2 ** 15, (rows, cols), generator=g).to(torch.int16)
        c = a.long() * b.long()

        def pt(t):
            rv, cv = (t.shape[0] - 1).bit_length(), (t.shape[1] - 1).bit_length()
            ref = TensorRef("committed", rv, cv, commitment=StubCommitment(rv + cv))
            return ProverTensor(None, ref, (), device=DeviceMatrix.from_int_tensor(t.cuda()))

        pr = zb.prove_elementprod(pt(a), pt(b), pt(c), StubKey(), tr, _Rng())
        return ([tuple(x.evaluations) for x in pr.sumcheck.rounds],
                tuple(pr.sumcheck.final_values), bytes(tr.state))
    d0 = d2 = n // 3
    d1 = n - 2 * d0
    a = torch.randint(-2 ** 15, 2 ** 15, (1 << d0, 1 << d1), generator=g).to(torch.int16).cuda()
    b = torch.randint(-2 ** 15, 2 ** 15, (1 << d1, 1 << d2), generator=g).to(torch.int16).cuda()
    c = torch.matmul(a.double(), b.double()).round().long()
    A, B, C = (DeviceMatrix.from_int_tensor(x) for x in (a, b, c))
    rounds, point, finals = zb.gadgets.matmul_sumcheck_replicated(A, B, C, (d0, d1, d2), tr)
    return rounds, tuple(finals), bytes(tr.state)


@pytest.mark.parametrize("world,kind,n", [(2, "elementprod", 22), (4, "elementprod", 22),
                                          (2, "zkmat_replicated", 22),
                                          (4, "zkmat_replicated", 22),
                                          (4, "range_lookup", 22)])
def test_sharded_gadgets_match_unsharded(kind, n, world):
    """prove_elementprod, the reference's dense zkMat claim and a quant_range
    lookup (sharded from 4 ranks: the dense Eq.-7 columns' shards), 2^22
    entries, with a ShardGroup active: the same proof as one GPU proving it
    alone (eq-factored / dense / tiled-indexed engines)."""
    import paper_2508_21393_b200 as zb

    res = _spawn(_gadget_worker, world, (kind, n))
    want = _gadget(kind, n, zb)
    for r in range(world):
        assert tuple(res[r]) == tuple(want), (kind, r)


@pytest.mark.parametrize("field,n", [("big", 16), ("test", 18)])
def test_sharded_engine_persistent_path_one_rank(field, n):
    """The persistent-engine branch of zkl_sumcheck_prove_sharded (the exchange
    inside run_phase's host round loop, what each rank runs on its own GPU),
    in a one-rank group: identical to run_rounds on the whole claim."""
    import paper_2508_21393_b200 as zb
    from paper_2508_21393_b200 import device as D
    from paper_2508_21393_b200 import shard
    from paper_2508_21393_b200.sumcheck import run_rounds

    p, tabs, terms, post_add, post_mul = _claim(field, n, 77 + n)
    spec = D.spec_for(p)
    out = []
    for sharded in (True, False):
        tr = zb.Transcript(b"shard1", p, b"seed")
        zb.sumcheck.absorb_claim(tr, 0, [zb.Term(c, f) for c, f in terms], 3, n)
        dev = [D.upload(t, spec) for t in tabs]
        if sharded:
            with shard.ShardGroup("p1" + secrets.token_hex(6), 0, 1):
                res = shard.run_rounds_sharded(spec, dev, n, terms, 3, tr, post_add=post_add,
                                               post_mul=post_mul)
        else:
            res = run_rounds(spec, dev, n, terms, 3, tr, post_add=post_add, post_mul=post_mul)
        out.append((res, bytes(tr.state)))
    assert out[0] == out[1]
