import sys, os, time
sys.path.insert(0, '.')
import torch
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import device as D, gadgets as G
from paper_2508_21393_b200.gadgets import DeviceMatrix
torch.cuda.set_device(0)
spec = D.spec_for(zb.MODULUS)
g = torch.Generator(device='cuda'); g.manual_seed(1)
cases = [("W 4096x4096 i16", torch.randint(-3000, 3000, (4096, 4096), device='cuda', dtype=torch.int16)),
         ("X 2048x4096 i16", torch.randint(-30000, 30000, (2048, 4096), device='cuda', dtype=torch.int16)),
         ("C 2048x4096 i64", torch.randint(-2**40, 2**40, (2048, 4096), device='cuda', dtype=torch.int64))]
for name, M in cases:
    Mx = DeviceMatrix.from_int_tensor(M)
    for tr in (False, True):
        n = M.shape[0] if tr else M.shape[1]
        x = D.eq_table([i * 7919 + 13 for i in range(n.bit_length() - 1)], spec)
        for _ in range(3): G._matvec(Mx, x, tr, spec)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): G._matvec(Mx, x, tr, spec)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        nbytes = M.numel() * M.element_size()
        print("%-18s %s %7.1f us  %6.0f GB/s" % (name, "M^T x" if tr else "M x  ", ms * 1e3, nbytes / ms / 1e6), flush=True)
