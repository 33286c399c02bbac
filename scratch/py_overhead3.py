import sys, time, cProfile, pstats
sys.path[:0] = ['.']
import torch, bench
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200.commit_stub import StubCommitment, StubKey
from paper_2508_21393_b200.gadgets import DeviceMatrix, ProverTensor, TensorRef
X, Y, tx, ty, logd = bench.cfg3_inputs()
class Pair:
    def __init__(s, x, y, name): s.x, s.y, s.name = x, y, name
pair = Pair(zb.LookupTable(tx, StubCommitment(16)), zb.LookupTable(ty, StubCommitment(16)), "silu")
def pt(t):
    ref = TensorRef("committed", logd // 2, logd - logd // 2, commitment=StubCommitment(logd))
    return ProverTensor(None, ref, (), device=DeviceMatrix.from_int_tensor(t))
class R:
    def vector(self, n): return [0] * n
def one(i):
    tr = zb.Transcript(b"cfg3", zb.MODULUS, b"%d" % i)
    return zb.prove_pair_lookup(b"swiglu/act", pt(X), pt(Y), pair, StubKey(), tr, R())
for i in range(3): one(i)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for i in range(5): one(10 + i)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
