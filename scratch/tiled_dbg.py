import sys
sys.path[:0] = ['.', 'tests']
import numpy as np
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import device as D, lookup as L
from paper_2508_21393_b200.commit_stub import StubCommitment, StubKey
from paper_2508_21393_b200.transcript import Transcript
from conftest import FIELDS
class R:
    def vector(self, n): return [0] * n
for field, d, n in [("test", 1 << 10, 1 << 5), ("big", 1 << 10, 1 << 5), ("big", 1 << 18, 1 << 12)]:
    p = FIELDS[field]; spec = D.spec_for(p)
    rnd = np.random.default_rng(d + n)
    table = [int(v) for v in rnd.integers(0, 2**40, size=n)]
    idx = rnd.integers(0, n, size=d)
    sec = D.upload([table[int(i)] for i in idx], spec)
    tab = zb.LookupTable(D.DeviceVector(D.upload(table, spec), n, spec), StubCommitment((n - 1).bit_length()))
    secret = zb.SecretVector(D.DeviceVector(sec, d, spec), StubCommitment((d - 1).bit_length()), ())
    out = []
    for tiled in (True, False):
        L.TILED = tiled
        m = zb.compute_multiplicities(secret.entries, tab)
        t = Transcript(b"tiled", p, b"x")
        pr = zb.prove_lookup(secret, m, tab, StubKey(), t, R())
        out.append([r.evaluations for r in pr.sumcheck.rounds])
    a, b = out
    bad = [(j, [x for x in range(4) if a[j][x] != b[j][x]]) for j in range(len(a)) if a[j] != b[j]]
    print(field, d, n, "rounds", len(a), "first bad", bad[:3])
    if bad:
        j = bad[0][0]
        for x in range(4):
            print("  x", x, a[j][x], b[j][x], (a[j][x] - b[j][x]) % p)
