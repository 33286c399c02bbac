import sys, time; sys.path.insert(0,'.'); sys.path.insert(0,'tests/golden')
import torch, ctypes
import bench
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import device as D, _native as N, sumcheck as S
from paper_2508_21393_b200.gadgets import DeviceMatrix
torch.cuda.set_device(0)
claims = bench.cfg2_claims(1234, 'cuda')
P = bench.P_BIG
spec = D.spec_for(P)
# warm
bench.prove_step(claims, 0, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
for name,a,b,c,dims in claims:
    tr = zb.Transcript(b"x", P, b"y")
    A,B,C = (DeviceMatrix.from_int_tensor(t) for t in (a,b,c))
    torch.cuda.synchronize(); t0=time.perf_counter()
    zb.matmul_sumcheck(A,B,C,dims,tr)
    torch.cuda.synchronize(); t1=time.perf_counter()
    print(name, dims, "%.2f ms"%((t1-t0)*1e3))
# per-round latency microbench: 2 tables of 2^12, 12 rounds via native driver
for n in (4, 8, 12, 16, 20):
    tabs=[D.upload(list(range(1,(1<<n)+1)), spec) for _ in range(2)]
    tr = zb.Transcript(b"x", P, b"y")
    torch.cuda.synchronize(); t0=time.perf_counter()
    for rep in range(5):
        tabs=[t.clone() for t in tabs]
        S.run_rounds(spec, tabs, n, [(1,(0,1))], 3, tr)
    torch.cuda.synchronize(); t1=time.perf_counter()
    print("n=%d: %.1f us/round" % (n, (t1-t0)*1e6/(5*n)))
# raw launch+sync latency
lib=N.lib()
x = torch.zeros(8, device='cuda')
torch.cuda.synchronize(); t0=time.perf_counter()
for i in range(1000):
    x.add_(1); torch.cuda.synchronize()
print("torch launch+sync: %.1f us" % ((time.perf_counter()-t0)*1e3))
