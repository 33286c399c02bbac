"""Host-side profile of resident cfg2 steps (cProfile): where the Python time
between the native zkMat calls goes."""
import cProfile
import pstats
import sys

sys.path[:0] = [".", "tests/golden"]
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_21393_b200 as zb  # noqa: E402
from paper_2508_21393_b200.gadgets import DeviceMatrix  # noqa: E402

torch.cuda.set_device(0)
claims = bench.cfg2_claims(1234, "cuda")
for s in range(3):
    bench.prove_step(claims, s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for s in range(10):
    bench.prove_step(claims, 10 + s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
