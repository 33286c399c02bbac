import sys, time
sys.path[:0] = ['.']
import torch, bench
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200.gadgets import DeviceMatrix
claims = bench.cfg2_claims(1234, 'cuda')
for s in range(3):
    bench.prove_step(claims, s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
t0 = time.perf_counter()
bench.prove_step(claims, 99, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
print("step ms %.3f" % ((time.perf_counter() - t0) * 1e3), file=sys.stderr)
