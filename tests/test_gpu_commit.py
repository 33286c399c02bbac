"""Hyrax row commitments on the GPU (paper_2508_21393_b200/commit_gpu.py,
csrc/commit.cu) against the Pedersen products computed with Python's pow in
both Schnorr groups (group.py:64-70), and against the reference's own
`commit` when baseline/_ref is installed."""

import os
import random
import sys
from collections import namedtuple

import pytest

from conftest import P_BIG, P_TEST

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2508_21393_b200 import commit_gpu  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
Group = namedtuple("Group", "q order cofactor")
Key = namedtuple("Key", "group generators blinding_generator seed max_vars")
GROUPS = {"big": Group(96 * P_BIG + 1, P_BIG, 96), "test": Group(52 * P_TEST + 1, P_TEST, 52)}


def _key(group, width, seed):
    rnd = random.Random(seed)

    def element():
        while True:
            e = pow(rnd.randrange(2, group.q - 1), group.cofactor, group.q)
            if e != 1:
                return e

    return Key(group, tuple(element() for _ in range(width)), element(), b"k%d" % seed, 30)


def _expected(key, table, num_vars, blinding):
    g, q = key.group, key.group.q
    rows, cols = commit_gpu._split_shape(num_vars)
    out = []
    for i in range(rows):
        acc = pow(key.blinding_generator, blinding[i], q) if blinding else 1
        for j in range(cols):
            acc = acc * pow(key.generators[j], table[i * cols + j], q) % q
        out.append(acc)
    return tuple(out)


@pytest.mark.parametrize("field", ["big", "test"])
@pytest.mark.parametrize("num_vars,blind", [(1, False), (6, True), (9, False), (9, True)])
def test_commit_rows_match_python_pow(field, num_vars, blind):
    group = GROUPS[field]
    p = group.order
    rows, cols = commit_gpu._split_shape(num_vars)
    key = _key(group, cols + 3, num_vars * 7 + len(field))
    rnd = random.Random(num_vars)
    table = [rnd.randrange(p) for _ in range(rows * cols)]
    specials = [0, 1, p - 1, 2, 255, 256, (1 << 64) % p, p - 32768, 32767]
    table[:len(specials)] = specials[:len(table)]
    blinding = [rnd.randrange(p) for _ in range(rows)] if blind else None
    got = commit_gpu.commit_rows(key, table, num_vars, blinding)
    assert got == _expected(key, table, num_vars, blinding)
    # the same table as a device vector (storage form, converted on the device)
    spec = D.spec_for(p)
    dv = D.DeviceVector(D.upload(table, spec), len(table), spec)
    assert commit_gpu.commit_rows(key, dv, num_vars, blinding) == got


def test_commit_rows_large_matches_python_on_sampled_rows():
    """A 2^16 table (256 rows x 256 columns): every row checked with pow on a
    sample of rows, and the int16-valued case (most bytes zero, negatives as
    p - |x|) the block's tensors commit."""
    group = GROUPS["big"]
    p = group.order
    num_vars = 16
    rows, cols = commit_gpu._split_shape(num_vars)
    key = _key(group, cols, 11)
    rnd = random.Random(3)
    table = [rnd.randrange(-32768, 32768) % p for _ in range(rows * cols)]
    got = commit_gpu.commit_rows(key, table, num_vars)
    q = group.q
    for i in (0, 1, 77, rows - 1):
        acc = 1
        for j in range(cols):
            acc = acc * pow(key.generators[j], table[i * cols + j], q) % q
        assert got[i] == acc, i


REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "zklora")),
                    reason="baseline/_ref not installed")
@pytest.mark.parametrize("field", ["big", "test"])
def test_commit_matches_reference_commit(field):
    """commit_gpu.commit against zklora.commit.commit with a real keygen key,
    binding-only and blinded."""
    sys.path.insert(0, REF)
    try:
        from zklora import commit as ref_commit
        from zklora import group as ref_group
    finally:
        sys.path.remove(REF)
    grp = ref_group.BIG_GROUP if field == "big" else ref_group.TEST_GROUP
    p = grp.order
    key = ref_commit.keygen(10, b"gpu-commit-test", grp)
    rnd = random.Random(5)
    table = [rnd.randrange(p) for _ in range(1 << 8)]
    assert commit_gpu.commit(key, table) == ref_commit.commit(key, table)
    blinding = [rnd.randrange(p) for _ in range(16)]
    assert commit_gpu.commit(key, table, blinding) == ref_commit.commit(key, table, blinding)


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "zklora")),
                    reason="baseline/_ref not installed")
def test_install_gpu_commit_proves_and_verifies_a_lookup():
    """install(gpu_commit=True) routes the reference's by-name `commit` to the
    GPU: a real-key prove_lookup (lookup.py:143-251, its m / A / B
    commitments on the GPU) verifies with the reference's verify_lookup."""
    sys.path.insert(0, REF)
    try:
        import zklora
        from zklora import commit as ref_commit
        from zklora import group as ref_group
        from zklora import lookup as ref_lookup
        from zklora.transcript import Transcript
    finally:
        sys.path.remove(REF)
    from paper_2508_21393_b200.install import install

    uninstall = install(zklora, gpu_commit=True)
    try:
        assert ref_lookup.commit.__wrapped__ is commit_gpu.commit
        p = P_BIG
        key = ref_commit.keygen(8, b"gpu-commit-lookup", ref_group.BIG_GROUP)
        rng = ref_commit.BlindingStream(b"blind", p)
        table = ref_lookup.make_lookup_table([v % p for v in range(-8, 8)], key)
        secret = ref_lookup.commit_secret([(i % 16 - 8) % p for i in range(32)], key, rng)
        counts = ref_lookup.compute_multiplicities(secret.entries, table)
        proof = ref_lookup.prove_lookup(secret, counts, table, key, Transcript(b"l", p, b"s"),
                                        rng)
        assert ref_lookup.verify_lookup(secret.commitment, table, proof, key,
                                        Transcript(b"l", p, b"s"))
    finally:
        uninstall()


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "zklora")),
                    reason="baseline/_ref not installed")
@pytest.mark.parametrize("field,num_vars,ntables", [("big", 7, 1), ("big", 10, 3), ("test", 9, 2)])
def test_open_batch_matches_reference(field, num_vars, ntables):
    """commit_gpu.open_batch against zklora.commit.open_batch on the same
    tables, point, transcript and blinding stream: the same values, the same
    OpeningProof, the same end transcript state, and verify_batch accepts."""
    sys.path.insert(0, REF)
    try:
        from zklora import commit as ref_commit
        from zklora import group as ref_group
        from zklora.transcript import Transcript
    finally:
        sys.path.remove(REF)
    grp = ref_group.BIG_GROUP if field == "big" else ref_group.TEST_GROUP
    p = grp.order
    key = ref_commit.keygen(num_vars, b"gpu-open-test", grp)
    rnd = random.Random(num_vars * 10 + ntables)
    rows, cols = ref_commit.split_shape(num_vars)
    tables = [[rnd.randrange(p) for _ in range(rows * cols)] for _ in range(ntables)]
    blindings = [[rnd.randrange(p) for _ in range(rows)] if k % 2 == 0 else None
                 for k in range(ntables)]
    point = [rnd.randrange(p) for _ in range(num_vars)]
    t1, t2 = Transcript(b"o", p, b"s"), Transcript(b"o", p, b"s")
    r1, r2 = ref_commit.BlindingStream(b"n", p), ref_commit.BlindingStream(b"n", p)
    want = ref_commit.open_batch(key, tables, blindings, point, t1, r1)
    got = commit_gpu.open_batch(key, tables, blindings, point, t2, r2)
    assert got == want
    assert t1.state == t2.state
    coms = [ref_commit.commit(key, t, b) for t, b in zip(tables, blindings)]
    assert ref_commit.verify_batch(key, coms, point, got[0], got[1], Transcript(b"o", p, b"s"))
