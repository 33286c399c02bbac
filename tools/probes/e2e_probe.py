import sys, time
sys.path[:0] = ['.']
import torch
import bench
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import device as D
from paper_2508_21393_b200.gadgets import DeviceMatrix
claims = bench.cfg2_claims(0, "cuda")
host = [(n, a.cpu().pin_memory(), b.cpu().pin_memory(), c.cpu().pin_memory(), d) for n, a, b, c, d in claims]
bufs = [(torch.empty_like(a, device="cuda"), torch.empty_like(b, device="cuda"), torch.empty_like(c, device="cuda")) for _, a, b, c, _ in host]
st = D.Staged()
def timed(fn, reps=5):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); out.append((time.perf_counter() - t0) * 1e3)
    return min(out), sum(out) / len(out)
for n, a, b, c, d in host:
    print(n, [tuple(x.shape) for x in (a, b, c)], [str(x.dtype) for x in (a, b, c)], sum(x.numel() * x.element_size() for x in (a, b, c)) / 1e6, "MB")
print("copies only (stream)", timed(lambda: st.stage([(a, b, c) for _, a, b, c, _ in host], out=bufs)))
print("copies only (default)", timed(lambda: [d_.copy_(h_, non_blocking=True) for hs, ds in zip(host, bufs) for h_, d_ in zip(hs[1:4], ds)]))
print("prove only", timed(lambda: bench.prove_step(claims, 1, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)))
def e2e():
    dev = st.stage([(a, b, c) for _, a, b, c, _ in host], out=bufs)
    sc = [(n, da, db, dc, d) for (n, _, _, _, d), (da, db, dc) in zip(host, dev)]
    bench.prove_step(sc, 2, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript, ready=st.ready)
print("e2e staged", timed(e2e))
# per-claim: when does each copy finish vs each proof
