"""Device time by kernel over one 7B LoRA-block proof (CUPTI via
torch.profiler): which kernels a block spends its GPU time in."""
import sys
import time

sys.path[:0] = [".", "tests/golden"]
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

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
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rec.replay(BK.BlockProver(zb.Transcript(b"b", P, b"x"), tables, timing=False))
    torch.cuda.synchronize()
wall = time.perf_counter() - t0
rows = sorted(((e.device_time_total, e.count, e.key) for e in prof.key_averages()
               if e.device_time_total > 0), reverse=True)
tot = sum(r[0] for r in rows)
print("wall %.3f s (under the profiler), device total %.3f s" % (wall, tot / 1e6))
for t, n, k in rows[:25]:
    print("%9.1f ms %6d  %5.1f%%  %s" % (t / 1e3, n, 100 * t / tot, k[:110]))
