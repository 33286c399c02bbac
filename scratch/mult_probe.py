import sys, time, ctypes
sys.path[:0] = ['.']
import torch, bench
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import lookup as L, device as D, _native as N
X, Y, tx, ty, logd = bench.cfg3_inputs()
spec = D.spec_for(zb.MODULUS)
alpha = 1234567891234567
tab = zb.LookupTable(D.pair_combine(tx, ty, alpha, spec), None)
sec = D.pair_combine(X, Y, alpha, spec)
def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3
print("pair total  %.3f ms" % t(lambda: L.multiplicities_pair(sec, tab, X, Y, tx, ty)))
print("indexed     %.3f ms" % t(lambda: L.multiplicities_indexed(sec, tab)))
print("range check %.3f ms" % t(lambda: torch.equal(tx.long(), torch.arange(int(tx[0]), int(tx[0]) + tx.numel(), device='cuda'))))
n = tx.numel(); d = len(sec)
tyi = ty.to(torch.int32).contiguous(); xs = X.contiguous().view(-1); ys = Y.contiguous().view(-1)
counts = torch.empty(n, dtype=torch.int32, device='cuda'); index = torch.empty(d, dtype=torch.int32, device='cuda')
fm = ctypes.c_int64(-1)
def call():
    N.check(N.lib().zkl_pair_multiplicities(spec.fid, D.ptr(xs), D._INT_TYPES[xs.dtype], D.ptr(ys), D._INT_TYPES[ys.dtype], d, int(tx[0]), D.ptr(tyi), D.ptr(sec.buf), D.ptr(tab.entries.buf), n, D.ptr(counts), D.ptr(index), ctypes.byref(fm), D.stream()))
print("C call      %.3f ms" % t(call))
