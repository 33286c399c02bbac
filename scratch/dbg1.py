import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests/golden')
import torch, numpy as np
from paper_2508_21393_b200 import device as D
from oracle import multilinear
P=D.MODULUS
for p in (D.MODULUS, D.TEST_MODULUS):
    spec=D.spec_for(p)
    vals=[0,1,-1,5,-300,2**40,-2**40, 2**62, -2**63, 2**63-1]
    t=torch.tensor(vals,dtype=torch.int64,device='cuda')
    got=D.download(D.lift(t,spec),spec,len(vals))
    print(p==P, got==[v%p for v in vals], got[:4])
    a=np.arange(-16,16).reshape(4,8)
    t=torch.from_numpy(a).cuda()
    buf=D.lift(t.view(-1),spec)
    pt=[3,5,7,11,13]
    from paper_2508_21393_b200.mle import mle_evaluate_device, mle_evaluate
    print(mle_evaluate_device(buf,5,pt,spec), multilinear.evaluate([int(x)%p for x in a.reshape(-1)],pt,p), mle_evaluate([int(x)%p for x in a.reshape(-1)],pt,p))
