"""Multi-GPU dense sumcheck: the boolean hypercube sharded across ranks.

SURVEY.md sec. 8e.  The reference binds the most-significant variable first
(mle.py:50-56), pairing global indices I and I + 2^(n-1) in round 0.  Ranks
therefore own tables CYCLICALLY on the low log2(G) index bits: rank g holds
the entries I = i*G + g (local index i), so every fold pair lives on one rank
and a round needs no table traffic at all:

  rounds 0 .. n-s-1 (s = log2 G): each rank folds + evaluates its shard, the
      (degree+1) partial evaluations are summed across ranks (one all-reduce
      of a few field elements), every rank appends the same evaluations to
      its own copy of the transcript and draws the same challenge;
  after n-s rounds each rank holds ONE entry per table (the folded table's
      entry g): an all-gather assembles the G-entry tables, which every rank
      finishes identically (the last s rounds).

Proofs are bit-identical to the unsharded prover for every G (tests:
tests/test_shard.py with gloo world_size 2 on CPU; tests/test_gpu_parity.py
simulates G = 2, 4, 8 shards on one GPU).

Field elements cross the collective as 16-bit limbs in int64 tensors, so a
plain SUM all-reduce (gloo or NCCL) is exact for any G < 2^47; the mod-p
reduction happens after the collective.
"""

import torch

from . import device as D

LIMBS = 16  # 16-bit limbs per element (covers both fields)


def to_limbs(values):
    """Python ints (< 2^256) -> int64 tensor of shape (len, 16)."""
    rows = [[(v >> (16 * i)) & 0xFFFF for i in range(LIMBS)] for v in values]
    return torch.tensor(rows, dtype=torch.int64).reshape(len(values), LIMBS)


def from_limbs(t, p):
    out = []
    for row in t.tolist():
        v = 0
        for i, limb in enumerate(row):
            v += int(limb) << (16 * i)
        out.append(v % p)
    return out


class Comm:
    """The collectives the sharded prover needs, over a torch.distributed
    process group (gloo or NCCL).  `device` is where the limb tensors live
    ("cpu" for gloo, "cuda" for NCCL)."""

    def __init__(self, group=None, device="cpu"):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.device = device
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def sum_mod(self, values, p):
        t = to_limbs(values).to(self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return from_limbs(t.cpu(), p)

    def gather(self, values, p):
        """-> list over ranks (rank order) of the value lists."""
        t = to_limbs(values).to(self.device)
        out = [torch.empty_like(t) for _ in range(self.size)]
        self.dist.all_gather(out, t, group=self.group)
        return [from_limbs(o.cpu(), p) for o in out]


class LocalComm:
    """G shards driven from ONE process (simulation on one device): the
    'collectives' are plain sums over the shard list, done on the host between
    rounds.  No kernel ever waits on another shard."""

    def __init__(self, size):
        self.size = size


def shard_of(values, rank, size):
    """Entries I = i*size + rank of a global table (cyclic low-bit sharding)."""
    return values[rank::size]


def prove_sharded(round_fn, finish_fn, num_vars, degree, terms, tr, comm, p,
                  post_add=None, post_mul=None, tail_fn=None):
    """Sharded sumcheck rounds after the claim is absorbed (sumcheck.py:108-130).

    round_fn(j, r_prev) -> this rank's raw evaluations (degree+1 canonical
        ints, no post scalars) for round j of its shard, folding by r_prev
        first when j > 0.
    finish_fn(r_last) -> this rank's k table entries folded by r_last (the
        one entry left after num_vars - s rounds).
    tail_fn(tables, rounds, point, post_add, post_mul) -> (rounds, point,
        finals) after the last s rounds over the gathered G-entry tables
        (device engine in production).
    Returns (rounds, point, finals) identical on every rank.
    """
    G = comm.size
    s = G.bit_length() - 1
    if G & (G - 1) or s >= num_vars:
        raise ValueError("shard count must be a power of two < 2^num_vars")
    rounds, point = [], []
    r_prev = None
    local_rounds = num_vars - s
    for j in range(local_rounds):
        raw = round_fn(j, r_prev)
        total = comm.sum_mod(raw, p)
        mul = 1 if post_mul is None else post_mul
        add = 0 if post_add is None else post_add[j]
        evals = tuple(mul * (v + add) % p for v in total)
        rounds.append(evals)
        for e in evals:
            tr.append(b"sumcheck/eval", e)
        r_prev = tr.challenge(b"sumcheck/round")
        point.append(r_prev)
    fin = finish_fn(r_prev)
    if isinstance(comm, LocalComm):
        per_rank = fin  # already one list per shard
    elif s == 0:
        return rounds, point, fin
    else:
        # one entry per table per rank: gather -> G-entry tables, finish the tail
        per_rank = comm.gather(fin, p)
    if s == 0:
        return rounds, point, per_rank[0]
    k = len(per_rank[0])
    tables = [[per_rank[g][t] for g in range(G)] for t in range(k)]
    tail_adds = post_add[local_rounds:] if post_add is not None else None
    return tail_fn(tables, rounds, point, tail_adds, post_mul)


# ---------------------------------------------------------------------------
# device round functions (one shard per rank, or G shards in one process)


class DeviceShard:
    """One shard of a claim on this rank's GPU, driven round by round through
    zkl_sumcheck_round (fused fold + evaluation, raw sums)."""

    def __init__(self, spec, tables, terms, degree):
        import ctypes

        from . import _native as N
        from .sumcheck import _TermArgs

        self.N, self.ctypes = N, ctypes
        self.spec, self.terms, self.degree = spec, terms, degree
        self.tables = tables
        self.size = tables[0].shape[0] if tables else 0
        self.ta = _TermArgs(terms, spec)
        self.ptrs = (ctypes.c_void_p * len(tables))(*[t.data_ptr() for t in tables])

    def round(self, j, r_prev):
        N, spec = self.N, self.spec
        nb = spec.nbytes
        buf = (self.ctypes.c_uint8 * (4 * nb))()
        rb = D.scalar_bytes(r_prev, spec) if j > 0 else None
        N.check(N.lib().zkl_sumcheck_round(spec.fid, self.ptrs, len(self.tables), self.size,
                                           1 if j > 0 else 0, rb, self.degree, self.ta.nt,
                                           self.ta.nf, self.ta.fi, self.ta.coeffs, None, None,
                                           buf, D.stream()))
        if j > 0:
            self.size //= 2
        return D.decode(bytes(buf), spec, self.degree + 1)

    def finish(self, r_last):
        N, spec = self.N, self.spec
        fin = (self.ctypes.c_uint8 * (len(self.tables) * spec.nbytes))()
        N.check(N.lib().zkl_sumcheck_finish(spec.fid, self.ptrs, len(self.tables),
                                            D.scalar_bytes(r_last, spec), fin, D.stream()))
        return D.decode(bytes(fin), spec, len(self.tables))


def device_tail(spec, terms, degree, tr):
    """tail_fn: the last s rounds over the gathered G-entry tables, on the
    device engine (run_rounds), appended to the rounds so far."""
    from .sumcheck import run_rounds

    def tail(tables, rounds, point, post_add, post_mul):
        dev = [D.upload(t, spec) for t in tables]
        n = (len(tables[0]) - 1).bit_length()
        r2, p2, fin = run_rounds(spec, dev, n, terms, degree, tr, post_add=post_add,
                                 post_mul=post_mul)
        return rounds + r2, point + p2, fin

    return tail


def prove_device_sharded(spec, local_tables, terms, degree, num_vars, tr, comm,
                         post_add=None, post_mul=None):
    """This rank's shard (local_tables: device field vectors of
    2^(num_vars - log2 G) entries, cyclic low-bit layout) through the sharded
    protocol; the claim must already be absorbed into `tr`."""
    sh = DeviceShard(spec, local_tables, terms, degree)
    return prove_sharded(sh.round, sh.finish, num_vars, degree, terms, tr, comm, spec.modulus,
                         post_add=post_add, post_mul=post_mul,
                         tail_fn=device_tail(spec, terms, degree, tr))


def prove_device_sharded_local(spec, global_tables, terms, degree, num_vars, tr, G,
                               post_add=None, post_mul=None):
    """G shards of one claim driven from this process on one GPU (each shard's
    rounds are independent launches; the per-round sums and the final gather
    are host-side).  Exercises exactly the sharded protocol of
    prove_device_sharded on a single device."""
    p = spec.modulus
    shards = []
    for g in range(G):
        loc = [t.view(-1, spec.words)[g::G].contiguous() for t in global_tables]
        shards.append(DeviceShard(spec, loc, terms, degree))

    class _Local(LocalComm):
        def sum_mod(self, values, p):  # values: list over shards
            return [sum(col) % p for col in zip(*values)]

        def gather(self, values, p):
            return values

    comm = _Local(G)

    def round_fn(j, r_prev):
        return [sh.round(j, r_prev) for sh in shards]

    def finish_fn(r_last):
        return [sh.finish(r_last) for sh in shards]

    return prove_sharded(round_fn, finish_fn, num_vars, degree, terms, tr, comm, p,
                         post_add=post_add, post_mul=post_mul,
                         tail_fn=device_tail(spec, terms, degree, tr))
