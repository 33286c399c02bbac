"""Host time of a resident cfg2 step outside the native zkMat call: wall time
of prove_step minus the time spent inside zkl_matmul_prove."""
import sys
import time

sys.path[:0] = [".", "tests/golden"]
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_21393_b200 as zb  # noqa: E402
from paper_2508_21393_b200 import _native as N  # noqa: E402
from paper_2508_21393_b200 import gadgets  # noqa: E402
from paper_2508_21393_b200.gadgets import DeviceMatrix  # noqa: E402

lib = N.lib()
inner = [0.0]


class Proxy:
    def __getattr__(self, name):
        f = getattr(lib, name)
        if name != "zkl_matmul_prove":
            return f

        def timed(*a):
            t0 = time.perf_counter()
            r = f(*a)
            inner[0] += time.perf_counter() - t0
            return r
        return timed


proxy = Proxy()
import types  # noqa: E402

fake = types.SimpleNamespace(**{k: getattr(N, k) for k in dir(N) if not k.startswith("__")})
fake.lib = lambda: proxy
gadgets.N = fake
torch.cuda.set_device(0)
claims = bench.cfg2_claims(1234, "cuda")
for s in range(3):
    bench.prove_step(claims, s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
inner[0] = 0.0
t0 = time.perf_counter()
K = 20
for s in range(K):
    bench.prove_step(claims, 10 + s, DeviceMatrix, zb.matmul_sumcheck, zb.Transcript)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print("wall ms/step %.3f  native ms/step %.3f  outside ms/step %.3f (%.1f us/claim)"
      % (wall / K * 1e3, inner[0] / K * 1e3, (wall - inner[0]) / K * 1e3,
         (wall - inner[0]) / K / 8 * 1e6))
