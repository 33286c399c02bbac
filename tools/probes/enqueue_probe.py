"""Host-side enqueue time of the witness product's pieces on a stream that is
blocked behind a long device sleep: any piece that synchronises shows up as
~the sleep length (diagnoses host stalls in the e2e step)."""
import sys
import time

sys.path[:0] = ["."]
import torch  # noqa: E402

from paper_2508_21393_b200 import device as D  # noqa: E402
from paper_2508_21393_b200 import _native as N  # noqa: E402

torch.cuda.set_device(0)
a = torch.randint(-300, 300, (2048, 4096), dtype=torch.int16, device="cuda")
b = torch.randint(-300, 300, (4096, 4096), dtype=torch.int16, device="cuda")
out = torch.empty((2048, 4096), dtype=torch.int64, device="cuda")
for _ in range(3):
    D.igemm16(a, b, out=out)
torch.cuda.synchronize()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    torch.cuda._sleep(2_000_000_000)  # ~1 s of device time on this stream
    t = time.perf_counter()
    ah = torch.empty((2048, 4096), dtype=torch.int8, device="cuda")
    al = torch.empty_like(ah)
    bh = torch.empty((4096, 4096), dtype=torch.int8, device="cuda")
    bl = torch.empty_like(bh)
    t1 = time.perf_counter()
    N.check(N.lib().zkl_split_i16(D.ptr(a), a.numel(), D.ptr(ah), D.ptr(al), D.stream()))
    t2 = time.perf_counter()
    hh = torch._int_mm(ah, bh)
    t3 = time.perf_counter()
    row = a.sum(1, dtype=torch.int64)
    t4 = time.perf_counter()
    c = D.igemm16(a, b, out=out)
    t5 = time.perf_counter()
    bt = torch.empty((4096, 4096), dtype=torch.int16, device="cuda")
    bt.copy_(b.t())
    t6 = time.perf_counter()
print("empty %.1f us, split %.1f us, _int_mm %.1f us, sum %.1f us, igemm16 %.1f us, "
      "transpose copy %.1f us" % ((t1 - t) * 1e6, (t2 - t1) * 1e6, (t3 - t2) * 1e6,
                                   (t4 - t3) * 1e6, (t5 - t4) * 1e6, (t6 - t5) * 1e6))
torch.cuda.synchronize()
