import sys, time, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests/golden')
import torch, bench
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import gadgets as G
from paper_2508_21393_b200.gadgets import DeviceMatrix
torch.cuda.set_device(0)
claims = bench.cfg2_claims(1234, 'cuda')
for native in (True, False):
    G.NATIVE_DRIVER = native
    for s in range(3):
        bench.prove_step(claims, s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
    torch.cuda.synchronize()
    ts = []
    for s in range(5):
        t0 = time.perf_counter()
        bench.prove_step(claims, 9 + s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print("native=%s step ms: %s" % (native, " ".join("%.2f" % (t * 1e3) for t in ts)), flush=True)
    # per claim
    for name, a, b, c, dims in claims:
        A, B, C = (DeviceMatrix.from_int_tensor(x) for x in (a, b, c))
        tr = zb.Transcript(b"x", bench.P_BIG, b"y")
        torch.cuda.synchronize(); t0 = time.perf_counter()
        zb.matmul_sumcheck(A, B, C, dims, tr)
        torch.cuda.synchronize()
        print("   %-10s %s %.3f ms" % (name, dims, (time.perf_counter() - t0) * 1e3), flush=True)
