import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests/golden')
import torch, numpy as np
from paper_2508_21393_b200 import device as D
from paper_2508_21393_b200.gadgets import DeviceMatrix, _matvec
P = D.MODULUS; spec = D.spec_for(P)
for dt in (torch.int16, torch.int64):
  for shape in [(2,4),(4,8),(1,1),(4,1),(1,8),(2,2),(8,32),(32,16),(4096,16),(16,4096),(2048,4096)]:
    for tr in (0,1):
        M = torch.randint(-1000, 1000, shape, dtype=torch.int64).to(dt).cuda()
        Md = DeviceMatrix.from_int_tensor(M)
        n = shape[0] if tr else shape[1]
        x = D.upload(list(range(1, n+1)), spec)
        y = _matvec(Md, x, bool(tr), spec)
        torch.cuda.synchronize()
        print(dt, shape, tr, "ok", flush=True)
