"""Sharded dense sumcheck: host-side protocol on CPU.

Two gloo ranks each own one cyclic low-bit shard of a seeded claim; the
per-round partial evaluations are all-reduced, the transcript runs on both
ranks, the last log2(G) rounds finish on the gathered tables.  The per-shard
round arithmetic here is the oracle's (test infrastructure); on the GPU the
same driver calls zkl_sumcheck_round (tests/test_gpu_parity.py).  The result
must equal the unsharded prover bit for bit, on both ranks.
"""

import os
import random
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import FIELDS
import inputs
from oracle import fs, sc
from oracle.multilinear import fold_msb
from paper_2508_21393_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _claim(field, n, k, seed):
    p = FIELDS[field]
    rnd = random.Random(seed)
    tabs = [inputs.field_vec(rnd.randrange(1 << 30), 1 << n, p) for _ in range(k)]
    terms = [(rnd.randrange(p), (0, 1, 2)), (rnd.randrange(p), (1,)), (rnd.randrange(p), (0, 2))]
    post_add = [rnd.randrange(p) for _ in range(n)]
    post_mul = rnd.randrange(p)
    return p, tabs, terms, post_add, post_mul


class _OracleShard:
    """Per-shard round arithmetic (oracle; CPU test stand-in for the device)."""

    def __init__(self, tables, terms, degree, p):
        self.t, self.terms, self.degree, self.p = [list(x) for x in tables], terms, degree, p

    def round(self, j, r_prev):
        if j > 0:
            self.t = [fold_msb(x, r_prev, self.p) for x in self.t]
        return sc.round_evals(self.t, self.terms, self.degree, self.p)

    def finish(self, r_last):
        return [fold_msb(x, r_last, self.p)[0] for x in self.t]


def _oracle_tail(terms, degree, p, tr):
    def tail(tables, rounds, point, post_add, post_mul):
        cur = [list(t) for t in tables]
        for j in range((len(cur[0]) - 1).bit_length()):
            ev = sc.round_evals(cur, terms, degree, p)
            mul = 1 if post_mul is None else post_mul
            add = 0 if post_add is None else post_add[j]
            ev = tuple(mul * (e + add) % p for e in ev)
            rounds.append(ev)
            for e in ev:
                tr.append(b"sumcheck/eval", e)
            r = tr.challenge(b"sumcheck/round")
            point.append(r)
            cur = [fold_msb(t, r, p) for t in cur]
        return rounds, point, [t[0] for t in cur]
    return tail


def _unsharded(p, tabs, terms, degree, n, post_add, post_mul):
    tr = fs.FS(b"shard", p, b"seed")
    sc.absorb_claim(tr, 0, terms, degree, n)
    cur = [list(t) for t in tabs]
    rounds, point = [], []
    for j in range(n):
        ev = sc.round_evals(cur, terms, degree, p)
        ev = tuple(post_mul * (e + post_add[j]) % p for e in ev)
        rounds.append(ev)
        for e in ev:
            tr.append(b"sumcheck/eval", e)
        r = tr.challenge(b"sumcheck/round")
        point.append(r)
        cur = [fold_msb(t, r, p) for t in cur]
    return rounds, point, [t[0] for t in cur], tr.state


def _worker(rank, world, port, field, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, tabs, terms, post_add, post_mul = _claim(field, n, 3, 11)
        tr = fs.FS(b"shard", p, b"seed")
        sc.absorb_claim(tr, 0, terms, 3, n)
        sh = _OracleShard([shard.shard_of(t, rank, world) for t in tabs], terms, 3, p)
        out = shard.prove_sharded(sh.round, sh.finish, n, 3, terms, tr, shard.Comm(), p,
                                  post_add=post_add, post_mul=post_mul,
                                  tail_fn=_oracle_tail(terms, 3, p, tr))
        q.put((rank, [list(r) for r in out[0]], out[1], list(out[2]), tr.state))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("field,n", [("test", 6), ("big", 5), ("test", 2)])
def test_sharded_world2_matches_unsharded(field, n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, field, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p, tabs, terms, post_add, post_mul = _claim(field, n, 3, 11)
    want = _unsharded(p, tabs, terms, 3, n, post_add, post_mul)
    for rank, rounds, point, finals, state in res:
        assert [tuple(r) for r in rounds] == want[0], rank
        assert point == want[1] and finals == want[2] and state == want[3], rank


def test_limb_codec_roundtrip():
    p = FIELDS["big"]
    vals = [0, 1, p - 1, 2**255 - 19, 12345678901234567890]
    t = shard.to_limbs(vals)
    assert shard.from_limbs(t, p) == [v % p for v in vals]
    # sums of G limb vectors stay exact
    s = shard.from_limbs(t * 8, p)
    assert s == [8 * v % p for v in vals]


def test_shard_layout_is_cyclic_low_bits():
    assert shard.shard_of(list(range(16)), 1, 4) == [1, 5, 9, 13]
