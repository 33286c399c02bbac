"""Deterministic commitment stub for commitment-free benchmarking and tests.

Commitments and openings are outside this backend's target (BASELINE.json:
"Polynomial commitment opening (Pedersen/Hyrax MSM) stays on the reference
path and is timed separately"), but their serialized bytes feed the
transcript.  With a real zklora CommitmentKey the prover delegates to
zklora.commit; with a StubKey it uses this stub, whose wire behaviour is
shared with oracle/stubcommit.py and tests/golden/make_golden.py:

  Commitment.serialize(group) = b"zkl-stub/v1" + u8(num_vars)
  open_batch appends each point coordinate (b"open/point") and each opened
  value (b"open/value") -- commit.py:192-195 -- and nothing else; the opened
  values are the true MLE evaluations (computed on the GPU).
"""

from dataclasses import dataclass, field, replace

STUB_TAG = b"zkl-stub/v1"

# Opening checks (harness/refverify.py): when True, stub commitments carry a
# handle on the data they stand for (a device tensor, or a recipe such as
# "1/(beta + s)" over one), so a checking verifier can evaluate the committed
# MLE independently of the prover and compare it with every opened value.
# Off in the product path: a handle keeps its tensor alive.
CHECK = False


@dataclass(frozen=True)
class StubCommitment:
    num_vars: int
    handle: object = field(default=None, compare=False, hash=False, repr=False)

    def serialize(self, group):
        return STUB_TAG + bytes([self.num_vars])


def attach(com, handle):
    """com with `handle` attached when CHECK is on (else com unchanged)."""
    if not CHECK or handle is None or not isinstance(com, StubCommitment):
        return com
    return replace(com, handle=handle)


class StubKey:
    """Stands in for zklora.commit.CommitmentKey (only .group is read)."""

    is_stub = True
    group = None


def split_shape(num_vars):
    """commit.py:26-29."""
    row_vars = (num_vars + 1) // 2
    return 1 << row_vars, 1 << (num_vars - row_vars)


def commit(key, table, blinding=None):
    return StubCommitment((len(table) - 1).bit_length())


def commit_size(num_vars):
    return StubCommitment(num_vars)


def combine_commitments(group, commitments, coefficients):
    handles = [getattr(c, "handle", None) for c in commitments]
    com = StubCommitment(commitments[0].num_vars)
    if any(h is None for h in handles):
        return com
    return attach(com, ("lin", list(zip(handles, coefficients))))


def open_batch(key, tables, blindings, point, tr, rng, values=None):
    """Stub opening; ``values`` may carry already-known evaluations."""
    if values is None:
        from .mle import mle_evaluate_many

        values = mle_evaluate_many(tables, point, tr.modulus)
    _append_all(tr, b"open/point", point)
    _append_all(tr, b"open/value", values)
    return list(values), None


def _append_all(tr, label, values):
    batch = getattr(tr, "append_ints", None)
    if batch is not None:
        batch(label, values)
    else:  # a foreign transcript (e.g. the reference's own)
        for v in values:
            tr.append(label, v)
