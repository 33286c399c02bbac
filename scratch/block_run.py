"""Prove one LLaMA-shaped LoRA block on cuda:0 and print the census."""
import json, sys, time
sys.path.insert(0, '.')
import torch
from paper_2508_21393_b200 import block as BK, device as D
from paper_2508_21393_b200.transcript import Transcript
P_BIG = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
shape = {"7b": BK.LLAMA2_7B, "13b": BK.LLAMA2_13B}[sys.argv[1] if len(sys.argv) > 1 else "7b"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
t0 = time.time()
tables = BK.block_tables(D.spec_for(P_BIG))
w = BK.BlockWitness(shape, seed=1)
torch.cuda.synchronize()
print("setup %.1f s" % (time.time() - t0), flush=True)
for i in range(reps):
    tr = Transcript(b"zklora-b200/block", P_BIG, b"%d" % i)
    torch.cuda.synchronize(); t0 = time.time()
    P = BK.prove_block(w, BK.BlockProver(tr, tables))
    torch.cuda.synchronize(); dt = time.time() - t0
    s = BK.summary(P)
    print("block %d: %.3f s, peak mem %.1f GB" % (i, dt, torch.cuda.max_memory_allocated() / 1e9), flush=True)
    print(json.dumps(s), flush=True)
