import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests/golden')
import torch, bench
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200.gadgets import DeviceMatrix
torch.cuda.set_device(0)
claims = bench.cfg2_claims(1234, 'cuda')
for s in range(2):
    bench.prove_step(claims, s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
bench.prove_step(claims, 9, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
