"""Host-side profile (cProfile) of one 7B LoRA-block proof replay: where the
Python time between native calls goes."""
import cProfile
import pstats
import sys
import time

sys.path[:0] = [".", "tests/golden"]
import torch  # noqa: E402

import paper_2508_21393_b200 as zb  # noqa: E402
from paper_2508_21393_b200 import block as BK  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402

P = D.MODULUS
tables = BK.block_tables(D.spec_for(P))
w = BK.BlockWitness(BK.LLAMA2_7B, seed=1)
rec = BK.prove_block(w, BK.WitnessRecorder(tables))
rec.replay(BK.BlockProver(zb.Transcript(b"b", P, b"w"), tables, timing=False))
torch.cuda.synchronize()
t0 = time.perf_counter()
rec.replay(BK.BlockProver(zb.Transcript(b"b", P, b"x"), tables, timing=False))
torch.cuda.synchronize()
print("block s (no profiler) %.3f" % (time.perf_counter() - t0))
pr = cProfile.Profile()
pr.enable()
rec.replay(BK.BlockProver(zb.Transcript(b"b", P, b"y"), tables, timing=False))
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(40)
st.sort_stats("cumulative").print_stats(40)
