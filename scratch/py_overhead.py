import sys, time
sys.path[:0] = ['.']
import torch, bench
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import _native as N, gadgets as G
from paper_2508_21393_b200.gadgets import DeviceMatrix
claims = bench.cfg2_claims(1234, 'cuda')
lib = N.lib()
orig = lib.zkl_matmul_prove
acc = [0.0]
class W:
    def __init__(s, f): s.f = f
    def __call__(s, *a):
        t0 = time.perf_counter(); r = s.f(*a); acc[0] += time.perf_counter() - t0; return r
lib.zkl_matmul_prove = W(orig)
for s in range(3):
    bench.prove_step(claims, s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
acc[0] = 0.0
t0 = time.perf_counter()
for s in range(10):
    bench.prove_step(claims, 100 + s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / 10
print("step %.3f ms, inside zkl_matmul_prove %.3f ms, outside %.3f ms" % (tot * 1e3, acc[0] / 10 * 1e3, (tot - acc[0] / 10) * 1e3))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for s in range(5):
    bench.prove_step(claims, 200 + s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
