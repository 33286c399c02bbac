"""Multi-GPU sharding, host side (CPU, no GPU): the native shared-memory
exchange that the sharded sumcheck engine runs between rounds
(paper_2508_21393_b200/csrc/shard.cu) as a real multi-process rank set --
all-gathers of varying payloads, thousands of back-to-back exchanges (the
two-slot tag protocol), and a process group opened from torch.distributed
(gloo) the way bench.py does under torchrun.  The device side (sharded
proofs equal to the unsharded prover) is tests/test_gpu_shard.py."""

import os
import secrets
import socket

import pytest
import torch.multiprocessing as mp


def _exchange_worker(rank, world, name, rounds, q):
    from paper_2508_21393_b200.shard import ShardGroup

    g = ShardGroup(name, rank, world)
    out = []
    for t in range(rounds):
        n = 1 + (t * 7) % 200  # equal across ranks for a given t
        payload = bytes(((rank * 31 + t + i) & 0xFF) for i in range(n))
        got = g.exchange(payload)
        ok = all(got[r] == bytes(((r * 31 + t + i) & 0xFF) for i in range(n))
                 for r in range(world))
        out.append(ok)
    g.close()
    q.put((rank, all(out)))


@pytest.mark.parametrize("world", [2, 4])
def test_native_exchange_all_gather(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = "t" + secrets.token_hex(6)
    ps = [ctx.Process(target=_exchange_worker, args=(r, world, name, 3000, q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dist_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2508_21393_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    with shard.ShardGroup.from_torch_distributed() as g:
        assert shard.active() is g and g.world == world
        got = g.exchange(b"rank%02d" % rank)
        q.put((rank, [x.decode() for x in got], shard.wants(22), shard.wants(12)))
    assert shard.active() is None
    dist.destroy_process_group()


def test_group_from_torch_distributed_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_dist_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=180) for _ in ps))
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        names, big, small = res[r]
        assert names == ["rank00", "rank01"] and big and not small
