"""Block proof profile: per-gadget times and lookup stage split."""
import collections, json, sys, time
sys.path.insert(0, '.')
import torch
from paper_2508_21393_b200 import block as BK, device as D, lookup as L, sumcheck as SC, gadgets as G, mle as M
from paper_2508_21393_b200.transcript import Transcript
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
prof = len(sys.argv) > 1 and sys.argv[1] == "stages"
if prof:
    for n in ("multiplicities_pair", "multiplicities_indexed", "batch_inverse_device", "_gather", "_expand", "_tiled_sumcheck", "run_rounds", "_finish_lookup"):
        wrap(L, n, "lookup." + n)
    wrap(D, "lift", "D.lift"); wrap(D, "pair_combine", "D.pair_combine")
    wrap(M, "mle_evaluate_matrix", "mle_matrix")
    import paper_2508_21393_b200.nonlinear as NL
    wrap(NL, "prove_pair_lookup", "pair_lookup(total)")
    wrap(G, "run_rounds", "elementprod.run_rounds"); wrap(G, "matmul_sumcheck", "matmul_sumcheck")
tables = BK.block_tables(D.spec_for(P_BIG))
w = BK.BlockWitness(BK.LLAMA2_7B, seed=1)
for i in range(2):
    T.clear()
    tr = Transcript(b"zklora-b200/block", P_BIG, b"%d" % i)
    torch.cuda.synchronize(); t0 = time.time()
    P = BK.prove_block(w, BK.BlockProver(tr, tables))
    torch.cuda.synchronize(); dt = time.time() - t0
print("block %.3f s  gadgets %.3f s  clipped %d" % (dt, sum(P.seconds), P.clipped))
rows = sorted(zip(P.seconds, P.log), key=lambda x: -x[0])
for sec, lg in rows[:40]:
    print("%8.2f ms  %s" % (sec * 1e3, lg))
agg = collections.defaultdict(lambda: [0, 0.0])
for sec, lg in zip(P.seconds, P.log):
    key = (lg[0], max(lg[1:]))
    agg[key][0] += 1; agg[key][1] += sec
print("--- by (kind, max rounds)")
for k, (c, sec) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print("%-22s n=%-3d %8.2f ms" % (k, c, sec * 1e3))
if prof:
    print("--- stages")
    for k, v in sorted(T.items(), key=lambda kv: -kv[1]):
        print("%-28s %8.2f ms" % (k, v * 1e3))
