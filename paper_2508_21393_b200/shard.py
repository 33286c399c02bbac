"""Multi-GPU dense sumcheck: the boolean hypercube sharded across the ranks of
one node (one process per GPU), SURVEY.md sec. 8e.

The reference binds the most-significant variable first (mle.py:50-56),
pairing global indices I and I + 2^(n-1) in round 0.  Ranks therefore own
tables CYCLICALLY on the low log2(G) index bits -- rank g holds the entries
I = i*G + g -- so every fold pair lives on one rank; the per-round exchange is
the (degree+1) partial evaluations, the last log2(G) rounds run on the
gathered one-entry-per-rank tables.  The engine is native
(zkl_sumcheck_prove_sharded, csrc/shard.cu): per round, the fused fold +
evaluation kernel on the shard, a host all-reduce through POSIX shared memory
(no Python, no device copies), the host transcript; proofs are the unsharded
prover's bit for bit, on every rank.

    with ShardGroup.from_torch_distributed():    # under torchrun
        prove_elementprod(...)                     # claims >= 2^SHARD_MIN_VARS shard

Which provers shard (when a group is active and the claim is large):
  prove_elementprod (gadgets.py:383-410): eq(r, .), A, B as cyclic shards;
  matmul_sumcheck_replicated (the reference's dense zkMat claim,
  gadgets.py:210-251; the cfg5 sweep): the replicated tables' shards, built
  from column slices of B and C (the low index bits are v's).
  prove_lookup (lookup.py:143-251, d >= n) from SHARD_LOOKUP_MIN_WORLD ranks:
  each rank materialises its shard of the seven Eq.-7 columns (the secret
  side gathered through the multiplicity index, the replicated table side
  as the table's own cyclic shard, tiled) and runs the dense evaluator.
Below that world size the single-GPU tiled logUp (eq-factored, table side
never replicated) does less work than a shard of the dense claim.
"""

import ctypes
import os
import secrets

from . import _native as N
from . import device as D

SHARD_MIN_VARS = 22  # below this a claim is latency-bound: one GPU proves it
# logUp with d >= n: a rank's shard of the dense 7-column claim costs ~20/G
# Montgomery products per query against ~8 on one GPU's tiled path (DESIGN.md
# sec. 4b), so lookups shard from 4 ranks up
SHARD_LOOKUP_MIN_WORLD = 4

_ACTIVE = None


class ShardGroup:
    """This process's membership in a rank set (one node, world a power of
    two).  Opening joins the shared-memory exchange region /zkl-<name>."""

    def __init__(self, name, rank, world):
        if world & (world - 1) or not 0 <= rank < world:
            raise ValueError("world must be a power of two and 0 <= rank < world")
        self.name, self.rank, self.world = name, rank, world
        N.check(N.load().zkl_shard_open(name.encode(), rank, world))
        self.open = True

    @classmethod
    def from_torch_distributed(cls, group=None):
        """One group per torch.distributed process group (rank 0 draws the
        region's name and broadcasts it)."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = [secrets.token_hex(8) + "-%d" % os.getpid() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        return cls(box[0], rank, world)

    def exchange(self, payload):
        """All-gather of one byte string per rank (equal lengths)."""
        out = (ctypes.c_uint8 * (len(payload) * self.world))()
        N.check(N.load().zkl_shard_exchange(payload, len(payload), out))
        n = len(payload)
        raw = bytes(out)
        return [raw[g * n:(g + 1) * n] for g in range(self.world)]

    def close(self):
        global _ACTIVE
        if self.open:
            N.check(N.load().zkl_shard_close())
            self.open = False
        if _ACTIVE is self:
            _ACTIVE = None

    def __enter__(self):
        global _ACTIVE
        _ACTIVE = self
        return self

    def __exit__(self, *exc):
        self.close()


def active():
    """The active ShardGroup with world > 1, or None."""
    g = _ACTIVE
    return g if g is not None and g.open and g.world > 1 else None


def wants(num_vars):
    """True when a claim of 2^num_vars entries should be sharded now."""
    g = active()
    return g is not None and num_vars >= SHARD_MIN_VARS and num_vars >= (g.world.bit_length())


def shard_of(t, spec, rank, world):
    """Entries I = i*world + rank of a device field vector (cyclic low-bit)."""
    return t.view(-1, spec.words)[rank::world].contiguous()


def eq_shard(point, spec, rank, world):
    """eq(point, I) for I = i*world + rank: eq(point_hi, i) * eq(point_lo, rank)
    (the low log2(world) coordinates pair with the rank bits, MSB first)."""
    from .mle import eq_eval

    s = world.bit_length() - 1
    n = len(point)
    p = spec.modulus
    bits = [(rank >> (s - 1 - b)) & 1 for b in range(s)]
    c = eq_eval(list(point[n - s:]), bits, p) if s else 1
    hi = D.eq_table(list(point[: n - s]), spec)
    out = D.empty(spec, 1 << (n - s))
    zero = D.empty(spec, 1 << (n - s)).zero_()
    N.check(N.lib().zkl_axpy(spec.fid, D.ptr(out), D.ptr(zero), D.scalar_bytes(c, spec),
                             D.ptr(hi), 1 << (n - s), D.stream()))
    return out


def run_rounds_sharded(spec, local_tables, num_vars, terms, degree, tr, post_add=None,
                       post_mul=None):
    """run_rounds (sumcheck.py) for this rank's shard of a claim of 2^num_vars
    entries (local tables: 2^(num_vars - log2 G) entries each, consumed): the
    same (rounds, point, finals) as the unsharded prover, on every rank."""
    from .sumcheck import _TermArgs, _decode, native_transcript

    if not native_transcript(tr, spec):
        raise ValueError("the sharded engine drives the native transcript")
    lib = N.lib()
    k = len(local_tables)
    ta = _TermArgs(terms, spec)
    ptrs = (ctypes.c_void_p * k)(*[t.data_ptr() for t in local_tables])
    nb = spec.nbytes
    addb = D.scalars_bytes(post_add, spec) if post_add is not None else None
    mulb = D.scalar_bytes(post_mul, spec) if post_mul is not None else None
    state = ctypes.create_string_buffer(bytes(tr.state), 64)
    rbuf = (ctypes.c_uint8 * (num_vars * (degree + 1) * nb))()
    pbuf = (ctypes.c_uint8 * (num_vars * nb))()
    fbuf = (ctypes.c_uint8 * (k * nb))()
    N.check(lib.zkl_sumcheck_prove_sharded(spec.fid, ptrs, k, num_vars, degree, ta.nt, ta.nf,
                                           ta.fi, ta.coeffs, addb, mulb, state, rbuf, pbuf, fbuf,
                                           D.stream()))
    flat = _decode(bytes(rbuf), nb, num_vars * (degree + 1))
    rounds = [tuple(flat[j * (degree + 1):(j + 1) * (degree + 1)]) for j in range(num_vars)]
    tr.state = state.raw[:64]
    log = getattr(tr, "log", None)
    if log is not None:
        log.extend((b"sumcheck/eval", (e.bit_length() + 7) // 8 or 1) for e in flat)
    return rounds, _decode(bytes(pbuf), nb, num_vars), _decode(bytes(fbuf), nb, k)
