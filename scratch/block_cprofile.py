"""cProfile of one LLaMA-2-7B block proof (host-side time split)."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import torch
from paper_2508_21393_b200 import block as BK, device as D
from paper_2508_21393_b200.transcript import Transcript
P_BIG = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
tables = BK.block_tables(D.spec_for(P_BIG))
w = BK.BlockWitness(BK.LLAMA2_7B, seed=1)
BK.prove_block(w, BK.BlockProver(Transcript(b"b", P_BIG, b"w"), tables))
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.time()
pr.enable()
BK.prove_block(w, BK.BlockProver(Transcript(b"b", P_BIG, b"x"), tables))
torch.cuda.synchronize()
pr.disable()
print("block %.3f s" % (time.time() - t0))
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
