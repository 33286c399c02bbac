"""Stage split of one range lookup (2^27 int16 secret) against the 2^16
quant_range and the 2^12 residue_range tables."""
import collections, sys, time
sys.path.insert(0, '.')
import torch
from paper_2508_21393_b200 import block as BK, device as D, lookup as L, nonlinear as NL
from paper_2508_21393_b200.transcript import Transcript
from paper_2508_21393_b200.gadgets import DeviceMatrix, ProverTensor, TensorRef
from paper_2508_21393_b200.commit_stub import StubCommitment, StubKey
P_BIG = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
T = collections.defaultdict(float)
def wrap(mod, name, label=None):
    f = getattr(mod, name)
    def w(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); T[label or name] += time.perf_counter() - t0
        return r
    setattr(mod, name, w)
for n in ("multiplicities_pair", "batch_inverse_device", "_gather", "_expand", "_tiled_sumcheck", "run_rounds", "_finish_lookup"):
    wrap(L, n)
wrap(D, "lift")
logd = int(sys.argv[1]) if len(sys.argv) > 1 else 27
tables = BK.block_tables(D.spec_for(P_BIG))
g = torch.Generator(device="cuda").manual_seed(1)
q = (torch.randn((1 << (logd - 11), 1 << 11), device="cuda", generator=g) * 5300).round().clamp(-32768, 32767).short()
r = torch.randint(-2048, 2048, q.shape, device="cuda", generator=g, dtype=torch.int32).short()
class R:
    def vector(self, n): return [0] * n
def pt(t):
    rv, cv = (t.shape[0] - 1).bit_length(), (t.shape[1] - 1).bit_length()
    return ProverTensor(None, TensorRef("committed", rv, cv, commitment=StubCommitment(rv + cv)), (), device=DeviceMatrix.from_int_tensor(t))
for name, t, tab in (("quant", q, tables.quant_range), ("resid", r, tables.residue_range)):
    for it in range(3):
        T.clear()
        tr = Transcript(b"x", P_BIG, b"%d" % it)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        NL._range_lookup(pt(t), tab, StubKey(), tr, R())
        torch.cuda.synchronize(); tot = time.perf_counter() - t0
    print("%s 2^%d: total %.2f ms" % (name, logd, tot * 1e3))
    for k, v in sorted(T.items(), key=lambda kv: -kv[1]):
        print("   %-24s %8.2f ms" % (k, v * 1e3))
