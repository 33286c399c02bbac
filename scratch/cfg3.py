"""cfg3 timing probe: SiLU pair lookup, 2^25 queries vs the 2^16 table."""
import base64, json, sys, time, zlib, os
sys.path[:0] = ['.', 'tests/golden']
import numpy as np, torch
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200.gadgets import DeviceMatrix, ProverTensor, TensorRef
from paper_2508_21393_b200.commit_stub import StubCommitment, StubKey
torch.cuda.set_device(0)
g = json.load(open('tests/golden/tables_g4096.json'))
ys = np.frombuffer(zlib.decompress(base64.b64decode(g["silu"]["y_zlib_b64"])), dtype="<i4")
x0 = g["silu"]["x0"]
tx = torch.arange(x0, x0 + len(ys), dtype=torch.int32, device='cuda')
ty = torch.from_numpy(ys.copy()).cuda()
logd = int(sys.argv[1]) if len(sys.argv) > 1 else 25
d = 1 << logd
nq = min(2048 * 11008, d)
rng = np.random.Generator(np.random.PCG64(7))
xq = np.clip(np.round(rng.normal(0, 1.5, nq) * 4096), -32768, 32767).astype(np.int32)
xs = np.zeros(d, dtype=np.int32); xs[:nq] = xq
ys_q = ys[xs - x0].astype(np.int32)  # padding rows: (0, silu(0) = 0)
X = torch.from_numpy(xs).cuda().view(1 << (logd // 2), -1)
Y = torch.from_numpy(ys_q).cuda().view(1 << (logd // 2), -1)
class PT:
    def __init__(s, x, y, name): s.x, s.y, s.name = x, y, name
pair = PT(zb.LookupTable(tx, StubCommitment(16)), zb.LookupTable(ty, StubCommitment(16)), "silu")
def ptens(t):
    ref = TensorRef("committed", logd // 2, logd - logd // 2, commitment=StubCommitment(logd))
    return ProverTensor(None, ref, (), device=DeviceMatrix.from_int_tensor(t))
key = StubKey()
class R:
    def vector(self, n): return [0] * n
for it in range(4):
    tr = zb.Transcript(b"cfg3", zb.MODULUS, b"%d" % it)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pr = zb.prove_pair_lookup(b"swiglu/act", ptens(X), ptens(Y), pair, key, tr, R())
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print("2^%d queries: %.3f s  rounds=%d retries=%d" % (logd, dt, len(pr.sumcheck.rounds), pr.beta_retries), flush=True)
