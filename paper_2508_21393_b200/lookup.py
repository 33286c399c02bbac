"""logUp lookup argument on the GPU (drop-ins for zklora.lookup).

prove_lookup follows lookup.py:143-251 step for step -- the same transcript
traffic, beta pole retries, Eq.-7 claim and openings -- with the heavy parts
on the device: beta + s and beta + t are inverted by one hierarchical
Montgomery-trick pass each (whose zero detection IS the pole test of
lookup.py:163-171), the seven lifted columns of lookup.py:188-202 are built
by zkl_expand, and the degree-3 sumcheck runs on the fused round engine.
When the secret is larger than the table the replicated table side is never
materialised: the first log2(d/n) rounds run with a tiled evaluator
(zkl_logup_tiled_rounds) and the rest over seven n-entry tables.
compute_multiplicities (lookup.py:91-99) is a device hash-table histogram.
"""

import ctypes
from dataclasses import dataclass

from . import _native as N
from . import device as D
from . import shard
from .field import batch_inverse_device, inverse_pow2
from .commit_stub import attach
from .gadgets import commit_backend
from .mle import mle_evaluate_device
from .sumcheck import TYPES as SC_TYPES
from .sumcheck import Term, absorb_claim, native_transcript, run_rounds

MAX_BETA_RETRIES = 3


class ElementNotInTable(ValueError):
    def __init__(self, index, value):
        super().__init__("secret entry %d (value %d) not in table" % (index, value))
        self.index = index
        self.value = value


class PoleCollision(RuntimeError):
    pass


@dataclass(frozen=True)
class LookupTable:
    entries: tuple
    commitment: object
    name: str = "table"

    @property
    def size(self):
        return len(self.entries)

    @property
    def num_vars(self):
        return (self.size - 1).bit_length()


@dataclass(frozen=True)
class SecretVector:
    entries: tuple
    commitment: object
    blinding: tuple

    @property
    def num_vars(self):
        return (len(self.entries) - 1).bit_length()


@dataclass
class LookupProof:
    secret_vars: int
    beta_retries: int
    multiplicity_commitment: object
    inverse_secret_commitment: object
    inverse_table_commitment: object
    sumcheck: object
    secret_values: tuple
    secret_opening: object
    table_values: tuple
    table_opening: object


TYPES = {"LookupProof": LookupProof, "ElementNotInTable": ElementNotInTable,
         "PoleCollision": PoleCollision}


def _terms(alpha, ratio, p):
    """lookup.py:116-126; factors 0 eq, 1 A, 2 S+beta, 3 ind, 4 B, 5 T+beta, 6 m."""
    a2 = alpha * alpha % p
    a3 = a2 * alpha % p
    return [
        Term(alpha, (0, 1, 2)),
        Term((-alpha) % p, (0, 3)),
        Term(a2, (0, 4, 5)),
        Term(a3, (1,)),
        Term((-a3 * ratio) % p, (6, 4)),
    ]


def _check_canonical(values, p, what):
    if values and (min(values) < 0 or max(values) >= p):
        raise NotImplementedError("%s must be canonical residues for the GPU path" % what)


def multiplicities_device(secret_buf, d, table_buf, n, spec, index=None):
    """Device histogram; returns (uint32 counts tensor, first_miss or None).
    `index` (int32 tensor of d entries) also receives each secret entry's
    table index."""
    import torch

    counts = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    fm = ctypes.c_int64(-1)
    if index is None:
        rc = N.lib().zkl_multiplicities(spec.fid, D.ptr(secret_buf), d, D.ptr(table_buf), n,
                                        D.ptr(counts), ctypes.byref(fm), D.stream())
    else:
        rc = N.lib().zkl_multiplicities_index(spec.fid, D.ptr(secret_buf), d, D.ptr(table_buf),
                                              n, D.ptr(counts), D.ptr(index), ctypes.byref(fm),
                                              D.stream())
    if rc == N.ZKL_ERR_MISSING:
        return counts, fm.value
    N.check(rc)
    return counts, None


def multiplicities_indexed(secret, table):
    """compute_multiplicities for device-resident entries, plus the table
    index of every secret entry (a uint32 device tensor of len(secret)).
    Raises ElementNotInTable like the reference (lookup.py:96-98)."""
    import torch

    spec = secret.spec
    sbuf = D.field_buffer(secret, spec)
    tbuf = D.field_buffer(table.entries, spec)
    d, n = len(secret), len(table.entries)
    index = torch.empty(max(d, 1), dtype=torch.int32, device="cuda")
    counts, miss = multiplicities_device(sbuf, d, tbuf, n, spec, index=index)
    if miss is not None:
        raise TYPES["ElementNotInTable"](miss, D.read_scalar(sbuf, spec, miss))
    out = D.empty(spec, n)
    N.check(N.lib().zkl_lift_u32(spec.fid, D.ptr(out), D.ptr(counts), n, D.stream()))
    return D.DeviceVector(out, n, spec), index


def multiplicities_pair(secret, table, x, y, tx, ty):
    """multiplicities_indexed for a pair lookup whose table x column is a
    consecutive integer range (tables.py:142-152): queries are binned from
    their int16/int32 (x, y) directly (zkl_pair_multiplicities).  Returns
    None when that does not apply (the caller then hashes combined values)."""
    import torch

    if x.dtype not in (torch.int16, torch.int32) or y.dtype not in (torch.int16, torch.int32):
        return None
    n = len(table.entries)
    tx = tx.reshape(-1)
    if tx.numel() != n or n == 0:
        return None
    x0 = int(tx[0])
    if not torch.equal(tx.long(), torch.arange(x0, x0 + n, device=tx.device)):
        return None
    ty = ty.reshape(-1).to(torch.int32).contiguous()
    spec = secret.spec
    tbuf = D.field_buffer(table.entries, spec)
    d = len(secret)
    xs = x.contiguous().view(-1)
    ys = y.contiguous().view(-1)
    counts = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    index = torch.empty(max(d, 1), dtype=torch.int32, device="cuda")
    fm = ctypes.c_int64(-1)

    def run(sbuf):
        return N.lib().zkl_pair_multiplicities(
            spec.fid, D.ptr(xs), D._INT_TYPES[xs.dtype], D.ptr(ys), D._INT_TYPES[ys.dtype], d, x0,
            D.ptr(ty), D.ptr(sbuf) if sbuf is not None else None, D.ptr(tbuf), n, D.ptr(counts),
            D.ptr(index), ctypes.byref(fm), D.stream())

    # a lazy PairColumn is binned from its integers first (no field buffer);
    # only a query off its table row needs the hash probe on x + alpha*y
    lazy = isinstance(secret, D.PairColumn) and not secret.materialized
    rc = run(None if lazy else D.field_buffer(secret, spec))
    if lazy and rc == N.ZKL_ERR_MISSING:
        rc = run(secret.buf)
    if rc == N.ZKL_ERR_UNSUPPORTED:
        return None
    if rc == N.ZKL_ERR_MISSING:
        value = (secret.value(fm.value) if isinstance(secret, D.PairColumn)
                 else D.read_scalar(D.field_buffer(secret, spec), spec, fm.value))
        raise TYPES["ElementNotInTable"](fm.value, value)
    N.check(rc)
    out = D.empty(spec, n)
    N.check(N.lib().zkl_lift_u32(spec.fid, D.ptr(out), D.ptr(counts), n, D.stream()))
    return D.DeviceVector(out, n, spec), index


def multiplicities_range(secret, table, col, tcol):
    """multiplicities_indexed for a single-column table whose entries are the
    consecutive integers tcol (quant_range / residue_range, tables.py:109-117)
    and a secret given by its signed int device column: bins by offset
    (zkl_range_multiplicities), never lifting the secret.  A secret entry
    outside the range is in no table entry: ElementNotInTable with the first
    such index, like lookup.py:96-98."""
    import torch

    if col.dtype not in (torch.int16, torch.int32, torch.int64):
        return None
    n = len(table.entries)
    x0 = int(tcol[0])
    spec = secret.spec
    xs = col.contiguous().view(-1)
    d = xs.numel()
    counts = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    index = torch.empty(max(d, 1), dtype=torch.int32, device="cuda")
    fm = ctypes.c_int64(-1)
    rc = N.lib().zkl_range_multiplicities(D.ptr(xs), D._INT_TYPES[xs.dtype], d, x0, n,
                                          D.ptr(counts), D.ptr(index), ctypes.byref(fm),
                                          D.stream())
    if rc == N.ZKL_ERR_MISSING:
        value = (secret.value(fm.value) if isinstance(secret, D.LiftedColumn)
                 else D.read_scalar(D.field_buffer(secret, spec), spec, fm.value))
        raise TYPES["ElementNotInTable"](fm.value, value)
    N.check(rc)
    out = D.empty(spec, n)
    N.check(N.lib().zkl_lift_u32(spec.fid, D.ptr(out), D.ptr(counts), n, D.stream()))
    return D.DeviceVector(out, n, spec), index


def _gather(spec, src, src_n, index, n, add=None):
    out = D.empty(spec, n)
    N.check(N.lib().zkl_gather(spec.fid, D.ptr(out), D.ptr(src), src_n, D.ptr(index), n,
                               D.scalar_bytes(add, spec) if add is not None else None,
                               D.stream()))
    return out


def compute_multiplicities(secret_entries, table, modulus=None):
    """Drop-in for zklora.lookup.compute_multiplicities (lookup.py:91-99).

    With device-resident entries (DeviceVector) the counts stay on the GPU
    and come back as a DeviceVector of field elements."""
    if isinstance(secret_entries, D.DeviceVector) or isinstance(table.entries, D.DeviceVector):
        spec = (secret_entries.spec if isinstance(secret_entries, D.DeviceVector)
                else table.entries.spec)
        sbuf = D.field_buffer(secret_entries, spec)
        tbuf = D.field_buffer(table.entries, spec)
        d, n = len(secret_entries), len(table.entries)
        counts, miss = multiplicities_device(sbuf, d, tbuf, n, spec)
        if miss is not None:
            raise TYPES["ElementNotInTable"](miss, D.read_scalar(sbuf, spec, miss))
        out = D.empty(spec, n)
        N.check(N.lib().zkl_lift_u32(spec.fid, D.ptr(out), D.ptr(counts), n, D.stream()))
        return D.DeviceVector(out, n, spec)
    entries = list(secret_entries)
    tab = list(table.entries)
    if modulus is None:
        from .field import MODULUS, TEST_MODULUS

        top = max(tab + entries + [0])
        modulus = TEST_MODULUS if top < TEST_MODULUS else MODULUS
    spec = D.spec_for(modulus)
    _check_canonical(entries, modulus, "secret entries")
    _check_canonical(tab, modulus, "table entries")
    sbuf = D.upload(entries, spec)
    tbuf = D.upload(tab, spec)
    counts, miss = multiplicities_device(sbuf, len(entries), tbuf, len(tab), spec)
    if miss is not None:
        raise TYPES["ElementNotInTable"](miss, entries[miss])
    return [int(c) for c in counts[: len(tab)].cpu().tolist()]


class _Sized:
    """len()-only stand-in handed to the commitment stub (no host copy)."""

    def __init__(self, n):
        self.n = n

    def __len__(self):
        return self.n


def _expand(spec, dst_n, src, src_n, mode, add=None, pad=None):
    out = D.empty(spec, dst_n)
    N.check(N.lib().zkl_expand(
        spec.fid, D.ptr(out), dst_n, D.ptr(src) if src is not None else None, src_n, mode,
        D.scalar_bytes(add, spec) if add is not None else None,
        D.scalar_bytes(pad, spec) if pad is not None else None, D.stream()))
    return out


def prove_lookup(secret, multiplicities, table, key, tr, rng, secret_index=None):
    """Drop-in for zklora.lookup.prove_lookup (lookup.py:143-251).

    secret_index (optional, from multiplicities_indexed): the table index of
    every secret entry.  The secret-side column 1/(beta + s_i) is then
    gathered from the table-side inversion instead of inverting d entries;
    since every s_i equals t_index(i), beta hits a secret pole only if it
    hits a table pole, so the retry decisions of lookup.py:163-171 are
    unchanged."""
    entries = secret.entries
    d, n = len(entries), table.size
    if d == 0 or d & (d - 1):
        raise ValueError("secret length must be a power of two")
    if len(multiplicities) != n:
        raise ValueError("multiplicity vector must match the table size")
    p = tr.modulus
    spec = D.spec_for(p)
    group = key.group
    be = commit_backend(key)
    stub = be.__name__.endswith("commit_stub")

    # m commitment + setup absorption (lookup.py:158-161)
    m_rows, _ = be.split_shape(table.num_vars)
    m_blinding = rng.vector(m_rows)
    m_commitment = be.commit(key, _Sized(n) if stub else D.as_list(multiplicities), m_blinding)
    if stub:  # (opening checks only: what m stands for, commit_stub.CHECK)
        m_commitment = attach(m_commitment, ("mult", entries, table.entries, multiplicities))
    tr.append(b"lookup/table", table.commitment.serialize(group))
    tr.append(b"lookup/secret", secret.commitment.serialize(group))
    tr.append(b"lookup/mult", m_commitment.serialize(group))

    # a LiftedColumn secret is only lifted when a path below needs the field
    # values (the indexed, tiled d >= n path never does)
    lazy = (isinstance(entries, (D.LiftedColumn, D.PairColumn)) and secret_index is not None
            and d >= n)
    s_buf = None if lazy else D.field_buffer(entries, spec)
    t_buf = D.field_buffer(table.entries, spec)
    m_buf = D.field_buffer(multiplicities, spec)

    # beta with pole retries (lookup.py:163-171): a pole is exactly a zero in
    # beta + s or beta + t, which the device batch inversion reports.
    retries = 0
    beta = tr.challenge(b"lookup/beta")
    while True:
        if secret_index is not None:
            z1 = None
            inv_t, z2 = batch_inverse_device(t_buf, n, spec, add=beta)
            inv_s = None  # gathered from inv_t on first use (the tiled path reads through the index)
        else:
            inv_s, z1 = batch_inverse_device(s_buf, d, spec, add=beta)
            z2 = None
            if z1 is None:
                inv_t, z2 = batch_inverse_device(t_buf, n, spec, add=beta)
        if z1 is None and z2 is None:
            break
        retries += 1
        if retries > MAX_BETA_RETRIES:
            raise TYPES["PoleCollision"]("challenge hit a pole %d times" % retries)
        tr.append(b"lookup/beta-retry", retries)
        beta = tr.challenge(b"lookup/beta")

    # helper-column commitments (lookup.py:175-180)
    a_rows, _ = be.split_shape(secret.num_vars)
    a_blinding = rng.vector(a_rows)
    def gathered_inv_s():
        return inv_s if inv_s is not None else _gather(spec, inv_t, n, secret_index, d)

    if stub:
        inv_s_host = inv_t_host = None
        a_commitment = attach(be.commit(key, _Sized(d), a_blinding), ("inv", entries, beta))
        b_commitment = attach(be.commit(key, _Sized(n)), ("inv", table.entries, beta))
    else:
        inv_s = gathered_inv_s()
        inv_s_host = D.download(inv_s, spec, d)
        inv_t_host = D.download(inv_t, spec, n)
        a_commitment = be.commit(key, inv_s_host, a_blinding)
        b_commitment = be.commit(key, inv_t_host)
    tr.append(b"lookup/inv-secret", a_commitment.serialize(group))
    tr.append(b"lookup/inv-table", b_commitment.serialize(group))

    alpha = tr.challenge(b"lookup/alpha")
    big = max(d, n)
    num_vars = (big - 1).bit_length()
    u = tr.challenge_vector(b"lookup/u", num_vars)
    ratio = inverse_pow2((big // n).bit_length() - 1, p)  # big / n is a power of two

    terms = _terms(alpha, ratio, p)
    claimed = alpha * alpha % p
    tuples = [(t.coefficient, t.factors) for t in terms]

    # multi-GPU (shard.py): with >= SHARD_LOOKUP_MIN_WORLD ranks every rank
    # materialises its cyclic shard of the seven Eq.-7 columns (1/G of the
    # replicated claim) and runs the dense logUp evaluator on it; below that
    # the single-GPU tiled path does less work than a shard of the dense claim
    g = shard.active()
    if (stub and g is not None and g.world >= shard.SHARD_LOOKUP_MIN_WORLD and d >= n >= g.world
            and shard.wants(num_vars) and native_transcript(tr, spec)):
        rounds, point, finals = _sharded_claim(spec, tr, g, d, n, s_buf, inv_s, t_buf, inv_t,
                                               m_buf, beta, u, terms, tuples, claimed, num_vars,
                                               secret_index, entries)
        return _finish_lookup(spec, p, key, be, stub, tr, rng, secret, table, multiplicities,
                              entries, beta, retries, m_commitment, a_commitment, b_commitment,
                              m_blinding, m_rows, a_blinding, inv_s, inv_s_host, inv_t_host,
                              s_buf, num_vars, rounds, point, finals, d, n)

    # secret larger than the table: the replicated table side (lookup.py:196-202)
    # is never materialised -- tiled rounds first, then 7 tables of n entries
    if d > n > 1 and TILED and native_transcript(tr, spec):
        tiled = _tiled_sumcheck(spec, tr, d, n, s_buf, inv_s, t_buf, inv_t, m_buf, beta, u,
                                terms, tuples, claimed, num_vars, secret_index)
        if tiled is not None:
            rounds, point, finals = tiled
            return _finish_lookup(spec, p, key, be, stub, tr, rng, secret, table, multiplicities,
                                  entries, beta, retries, m_commitment, a_commitment, b_commitment,
                                  m_blinding, m_rows, a_blinding, inv_s, inv_s_host, inv_t_host,
                                  s_buf, num_vars, rounds, point, finals, d, n)

    if s_buf is None:
        s_buf = D.field_buffer(entries, spec)
    inv_s = gathered_inv_s()
    # lifted columns (lookup.py:188-202)
    if d <= n:
        A = _expand(spec, n, inv_s, d, 0)
        Sb = _expand(spec, n, s_buf, d, 0, add=beta, pad=beta)
        ind = _expand(spec, n, None, d, 0, add=1, pad=0)
        Bt = inv_t.clone()
        Tb = _expand(spec, n, t_buf, n, 1, add=beta)
        Mt = m_buf.clone()
    else:
        A = inv_s.clone()
        Sb = _expand(spec, d, s_buf, d, 1, add=beta)
        ind = _expand(spec, d, None, d, 0, add=1, pad=0)
        Bt = _expand(spec, d, inv_t, n, 1)
        Tb = _expand(spec, d, t_buf, n, 1, add=beta)
        Mt = _expand(spec, d, m_buf, n, 1)
    E = D.eq_table(u, spec)
    absorb_claim(tr, claimed, terms, 3, num_vars)
    if num_vars:
        rounds, point, finals = run_rounds(spec, [E, A, Sb, ind, Bt, Tb, Mt], num_vars, tuples,
                                           3, tr)
    else:
        rounds, point = [], []
        finals = [D.read_scalar(x, spec) for x in (E, A, Sb, ind, Bt, Tb, Mt)]
    return _finish_lookup(spec, p, key, be, stub, tr, rng, secret, table, multiplicities, entries,
                          beta, retries, m_commitment, a_commitment, b_commitment, m_blinding,
                          m_rows, a_blinding, inv_s, inv_s_host, inv_t_host, s_buf, num_vars,
                          rounds, point, finals, d, n)


TILED = True  # tests flip this to compare with the fully materialised claim


def _sharded_claim(spec, tr, g, d, n, s_buf, inv_s, t_buf, inv_t, m_buf, beta, u, terms,
                   tuples, claimed, num_vars, secret_index, entries):
    """This rank's cyclic shard (global entries i = i' G + rank) of the Eq.-7
    claim's seven columns for d >= n (lookup.py:196-202: the table side
    replicated d / n times), proven through the sharded engine.  Global entry
    i's table index is i mod n, which is congruent to the rank mod G, so the
    replicated table columns are the table's own cyclic shard, tiled."""
    G, rk = g.world, g.rank
    W = spec.words
    dl, nl = d // G, n // G
    E = shard.eq_shard(u, spec, rk, G)
    Tb_full = _expand(spec, n, t_buf, n, 1, add=beta)
    if secret_index is not None:  # every s_i is the table entry at its index
        idx = secret_index[:d][rk::G].contiguous()
        A = _gather(spec, inv_t, n, idx, dl)
        Sb = _gather(spec, Tb_full, n, idx, dl)
    else:
        sb = s_buf if s_buf is not None else D.field_buffer(entries, spec)
        A = inv_s.view(-1, W)[:d][rk::G].contiguous()
        Sb = _expand(spec, dl, sb.view(-1, W)[:d][rk::G].contiguous(), dl, 1, add=beta)
    ind = _expand(spec, dl, None, dl, 0, add=1, pad=0)

    def tiled(col):
        return _expand(spec, dl, col.view(-1, W)[:n][rk::G].contiguous(), nl, 1)

    Bt, Tb, Mt = tiled(inv_t), tiled(Tb_full), tiled(m_buf)
    absorb_claim(tr, claimed, terms, 3, num_vars)
    return shard.run_rounds_sharded(spec, [E, A, Sb, ind, Bt, Tb, Mt], num_vars, tuples, 3, tr)


def _tiled_sumcheck(spec, tr, d, n, s_buf, inv_s, t_buf, inv_t, m_buf, beta, u, terms, tuples,
                    claimed, num_vars, secret_index=None):
    """zkl_logup_tiled_rounds for the high log2(d/n) variables (the replicated
    table side and the eq table are never materialised), then the remaining
    log2(n) rounds over 7 tables of n entries (indicator = ones).  Returns
    None (nothing consumed, transcript untouched) when the native engine
    declines (stepwise mode under profilers, n < 32)."""
    tile_log = (n - 1).bit_length()
    r1 = num_vars - tile_log
    # indexed: A_i = 1/(beta + t_idx(i)) and S_i = t_idx(i) + beta are read
    # through the index in rounds 0-1 and never materialised; the first fold
    # writes d/2-entry tables
    indexed = secret_index is not None and r1 >= 2
    Tb = _expand(spec, n, t_buf, n, 1, add=beta)
    if indexed:
        A = D.empty(spec, d // 2)
        Sb = D.empty(spec, d // 2)
    else:
        # inv_s / inv_t are consumed in place: with d > n the openings use the
        # sumcheck finals, and the commitment path downloaded them already
        A = inv_s if inv_s is not None else _gather(spec, inv_t, n, secret_index, d)
        if secret_index is not None:  # s_i + beta == t_index(i) + beta
            Sb = _gather(spec, Tb, n, secret_index, d)
        else:
            Sb = _expand(spec, d, s_buf, d, 1, add=beta)
    Bb = inv_t
    Mb = m_buf.clone()  # may be the caller's DeviceVector buffer
    E = D.empty(spec, n)
    nb = spec.nbytes
    before = bytes(tr.state)
    absorb_claim(tr, claimed, terms, 3, num_vars)
    state = ctypes.create_string_buffer(bytes(tr.state), 64)
    rbuf = (ctypes.c_uint8 * (r1 * 4 * nb))()
    pbuf = (ctypes.c_uint8 * (r1 * nb))()
    ptrs = (ctypes.c_void_p * 7)(*[t.data_ptr() for t in (E, A, Sb, Bb, Tb, Mb)],
                                 secret_index.data_ptr() if indexed else None)
    coeffs = D.scalars_bytes([t.coefficient for t in terms], spec)
    ub = D.scalars_bytes(list(u), spec)
    rc = N.lib().zkl_logup_tiled_rounds(spec.fid, ptrs, tile_log, num_vars, r1, ub, coeffs,
                                        1 | (2 if indexed else 0), state, rbuf, pbuf,
                                        D.stream())
    if rc == N.ZKL_ERR_UNSUPPORTED:
        tr.state = before
        log = getattr(tr, "log", None)
        if log is not None:
            del log[-(2 + 2 * len(terms)):]
        return None
    N.check(rc)
    flat = D.decode(bytes(rbuf), spec, 4 * r1)
    rounds = [tuple(flat[4 * j:4 * j + 4]) for j in range(r1)]
    point = D.decode(bytes(pbuf), spec, r1)
    tr.state = state.raw[:64]
    log = getattr(tr, "log", None)
    if log is not None:
        log.extend((b"sumcheck/eval", (e.bit_length() + 7) // 8 or 1) for e in flat)
    ind = _expand(spec, n, None, n, 0, add=1, pad=0)
    r2, p2, finals = run_rounds(spec, [E, A[:n], Sb[:n], ind, Bb, Tb, Mb], tile_log, tuples,
                                3, tr)
    return rounds + r2, point + p2, finals


def _finish_lookup(spec, p, key, be, stub, tr, rng, secret, table, multiplicities, entries, beta,
                   retries, m_commitment, a_commitment, b_commitment, m_blinding, m_rows,
                   a_blinding, inv_s, inv_s_host, inv_t_host, s_buf, num_vars, rounds, point,
                   finals, d, n):
    RP = SC_TYPES["RoundPolynomial"]
    sc_proof = SC_TYPES["SumcheckProof"]([RP(e) for e in rounds], tuple(finals))

    # openings (lookup.py:221-239)
    d_vars, n_vars = secret.num_vars, table.num_vars
    secret_point = point[num_vars - d_vars:]
    table_point = point[num_vars - n_vars:]
    zero_blind = [0] * m_rows
    if stub:
        if d >= n:  # finals are the unpadded MLEs (replication is MLE-transparent)
            s_vals = [finals[1], (finals[2] - beta) % p]
        else:
            s_vals = [mle_evaluate_device(inv_s, d_vars, secret_point, spec),
                      mle_evaluate_device(s_buf, d_vars, secret_point, spec)]
        # the table side is either unpadded (d <= n) or replicated (d > n)
        t_vals = [finals[6], finals[4], (finals[5] - beta) % p]
        secret_values, secret_opening = be.open_batch(
            key, None, None, secret_point, tr, rng, values=s_vals)
        table_values, table_opening = be.open_batch(
            key, None, None, table_point, tr, rng, values=t_vals)
    else:
        secret_values, secret_opening = be.open_batch(
            key, [inv_s_host, D.as_list(entries)], [list(a_blinding), list(secret.blinding)],
            secret_point, tr, rng)
        table_values, table_opening = be.open_batch(
            key, [D.as_list(multiplicities), inv_t_host, D.as_list(table.entries)],
            [list(m_blinding), zero_blind, zero_blind], table_point, tr, rng)
    return TYPES["LookupProof"](
        secret.num_vars, retries, m_commitment, a_commitment, b_commitment, sc_proof,
        tuple(secret_values), secret_opening, tuple(table_values), table_opening)
