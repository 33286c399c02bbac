"""Fiat-Shamir transcript (oracle restatement).

Follows /root/reference/pkg/src/zklora/transcript.py:13-53: a 64-byte
rolling SHAKE-256 state; records are framed as
u16le(len label) | label | u64le(len data) | data; ints are appended in
minimal little-endian form (at least one byte); a challenge squeezes 64
bytes, re-absorbs them under the label "drawn", and reduces mod p.
"""

import hashlib


def record(label, payload):
    return b"".join(
        (len(label).to_bytes(2, "little"), label, len(payload).to_bytes(8, "little"), payload)
    )


def int_bytes(v):
    return v.to_bytes(max(1, (v.bit_length() + 7) // 8), "little")


def _h(data):
    return hashlib.shake_256(data).digest(64)


class FS:
    def __init__(self, domain, p, seed=b""):
        self.modulus = p
        self.state = _h(record(b"domain", domain) + record(b"seed", seed))
        self.log = []

    def append(self, label, data):
        if isinstance(data, int):
            data = int_bytes(data)
        self.log.append((label, len(data)))
        self.state = _h(self.state + record(label, data))

    def challenge(self, label):
        raw = _h(self.state + record(b"challenge", label))
        self.state = _h(self.state + record(b"drawn", raw))
        return int.from_bytes(raw, "little") % self.modulus

    def challenge_vector(self, label, count):
        out = []
        for k in range(count):
            out.append(self.challenge(label + b"/" + str(k).encode()))
        return out
