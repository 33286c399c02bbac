"""One traced cfg2 step (ZKL_TRACE=1 must be set): per claim, the GPU time
of each segment of the zkMat driver (csrc/zkmat.cu) and the host marks."""
import sys
import time

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
print("---- traced step", file=sys.stderr, flush=True)
t0 = time.perf_counter()
bench.prove_step(claims, 9, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
print("step wall ms %.3f" % ((time.perf_counter() - t0) * 1e3), file=sys.stderr)
