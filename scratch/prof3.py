import sys, time; sys.path.insert(0,'.')
import torch
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import device as D, sumcheck as S
torch.cuda.set_device(0)
P = zb.MODULUS; spec = D.spec_for(P)
for n in (4, 12, 20):
  for k, terms in ((2, [(1,(0,1))]), (7, [(3,(0,1,2)),(5,(0,3)),(7,(0,4,5)),(9,(1,)),(11,(6,4))])):
    tabs=[D.upload(list(range(1,(1<<n)+1)), spec) for _ in range(k)]
    tr = zb.Transcript(b"x", P, b"y")
    for rep in range(2):
        tt=[t.clone() for t in tabs]
        torch.cuda.synchronize(); t0=time.perf_counter()
        S.run_rounds(spec, tt, n, terms, 3, tr)
        torch.cuda.synchronize(); t1=time.perf_counter()
    print("n=%d k=%d: %.1f us/round" % (n, k, (t1-t0)*1e6/n), flush=True)
