"""Deterministic commitment stub (test / benchmark infrastructure).

Commitments and openings are outside this repo's target (BASELINE.json
north star; SURVEY.md sec. 8c "Parity at scale").  Their serialized bytes
still feed the transcript, so parity runs install the SAME stub on both
sides: on the reference (monkeypatching zklora.lookup / zklora.gadgets
``commit`` and ``open_batch`` in tests/golden/make_golden.py) and on the
product (``paper_2508_21393_b200.commit_stub``).

Wire format (must match paper_2508_21393_b200/commit_stub.py):
  commitment.serialize(group) = b"zkl-stub/v1" + u8(num_vars)
  open_batch: appends every point coordinate under b"open/point" and every
  opened value under b"open/value" (commit.py:192-195), nothing else; the
  opened values are the true MLE evaluations.
"""

from .multilinear import evaluate

STUB_TAG = b"zkl-stub/v1"


def stub_bytes(num_vars):
    return STUB_TAG + bytes([num_vars])


class StubBackend:
    """Backend object for oracle.logup: commit -> bytes, open -> values."""

    def __init__(self, p):
        self.p = p

    def commit(self, table):
        return stub_bytes((len(table) - 1).bit_length())

    def open(self, tables, point, tr):
        vals = [evaluate(t, point, self.p) for t in tables]
        for r in point:
            tr.append(b"open/point", r)
        for y in vals:
            tr.append(b"open/value", y)
        return vals

    def check(self, values, point, tr):
        for r in point:
            tr.append(b"open/point", r)
        for y in values:
            tr.append(b"open/value", y)
        return True
