"""Per-phase wall breakdown of one cfg2 bench step (host timers, synced)."""
import sys, time, collections, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests/golden')
import torch, bench
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import gadgets as G, sumcheck as S, device as D
from paper_2508_21393_b200.gadgets import DeviceMatrix
torch.cuda.set_device(0)
claims = bench.cfg2_claims(1234, 'cuda')
for s in range(3):
    bench.prove_step(claims, s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
acc = collections.defaultdict(float); cnt = collections.Counter()
def wrap(mod, name, key):
    f = getattr(mod, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); acc[key] += time.perf_counter() - t; cnt[key] += 1
        return r
    setattr(mod, name, g)
wrap(G, '_matvec', 'matvec'); wrap(G, 'run_rounds', 'run_rounds'); wrap(D, 'eq_table', 'eq_table')
wrap(D, 'dot', 'dot'); wrap(G, '_axpy', 'axpy')
torch.cuda.synchronize(); t0 = time.perf_counter()
bench.prove_step(claims, 9, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize(); tot = time.perf_counter() - t0
for k in acc: print("%-12s n=%3d %8.3f ms" % (k, cnt[k], acc[k] * 1e3))
print("total %.3f ms, other %.3f ms" % (tot * 1e3, (tot - sum(acc.values())) * 1e3))
# unwrapped timing
for f in ('_matvec', 'run_rounds'):
    pass
