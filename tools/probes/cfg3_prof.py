"""cfg3 stage breakdown: wraps the lookup stages with synchronising timers."""
import sys, time, collections
sys.path[:0] = ['.']
import torch
import bench
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import lookup as L, device as D, gadgets as G, sumcheck as SC, field as FLD
from paper_2508_21393_b200.commit_stub import StubCommitment, StubKey
from paper_2508_21393_b200.gadgets import DeviceMatrix, ProverTensor, TensorRef
T = collections.defaultdict(float)
def wrap(mod, name, label=None):
    f = getattr(mod, name)
    def w(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); T[label or name] += time.perf_counter() - t0
        return r
    setattr(mod, name, w)
wrap(D, "pair_combine")
wrap(L, "multiplicities_indexed"); wrap(L, "multiplicities_pair")
wrap(L, "batch_inverse_device")
wrap(L, "_gather"); wrap(L, "_expand"); wrap(L, "_tiled_sumcheck"); wrap(L, "run_rounds"); wrap(L, "_finish_lookup")
wrap(L, "absorb_claim")
X, Y, tx, ty, logd = bench.cfg3_inputs()
class Pair:
    def __init__(s, x, y, name): s.x, s.y, s.name = x, y, name
pair = Pair(zb.LookupTable(tx, StubCommitment(16)), zb.LookupTable(ty, StubCommitment(16)), "silu")
def pt(t):
    ref = TensorRef("committed", logd // 2, logd - logd // 2, commitment=StubCommitment(logd))
    return ProverTensor(None, ref, (), device=DeviceMatrix.from_int_tensor(t))
class R:
    def vector(self, n): return [0] * n
for it in range(5):
    if it == 2: T.clear()
    tr = zb.Transcript(b"cfg3", zb.MODULUS, b"%d" % it)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pr = zb.prove_pair_lookup(b"swiglu/act", pt(X), pt(Y), pair, StubKey(), tr, R())
    torch.cuda.synchronize(); T["TOTAL"] += time.perf_counter() - t0
for k, v in sorted(T.items(), key=lambda kv: -kv[1]):
    print("%-28s %8.3f ms" % (k, v / 3 * 1e3))
