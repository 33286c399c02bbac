import sys, random, time
sys.path[:0] = ['.', 'tests', 'tests/golden']
import torch
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import device as D, sumcheck as S
torch.cuda.set_device(0)
p = zb.MODULUS
spec = D.spec_for(p)
field = sys.argv[2] if len(sys.argv) > 2 else 'big'
if field == 'test': p = zb.TEST_MODULUS; spec = D.spec_for(p)
n = int(sys.argv[1])
terms = [(5, (0, 1, 2)), (p - 5, (0, 3)), (7, (0, 4, 5)), (9, (1,)), (p - 11, (6, 4))]
tabs = []
for j in range(7):
    t = D.empty(spec, 1 << n)
    t.random_(0, 2**62)
    if spec.words == 4:
        t[:, 3] &= (1 << 60) - 1
    else:
        t[:, 0] &= (1 << 60) - 1
    tabs.append(t)
tr = zb.Transcript(b"x", p, b"y")
t0 = time.time()
try:
    r = S.run_rounds(spec, tabs, n, terms, 3, tr)
    print("n=%d %s ok %.3f s" % (n, field, time.time() - t0))
except Exception as e:
    print("n=%d %s FAIL %s (%.1f s)" % (n, field, e, time.time() - t0))
