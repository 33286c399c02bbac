"""GPU timeline of one resident cfg2 step through torch.profiler (CUPTI sees
every kernel, the library's included): per claim, each kernel's start, length
and the idle gap before it; written to gpurun_out/timeline/."""
import json
import os
import sys

sys.path[:0] = [".", "tests/golden"]
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2508_21393_b200 as zb  # noqa: E402
from paper_2508_21393_b200.gadgets import DeviceMatrix  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline"
os.makedirs(out, exist_ok=True)
torch.cuda.set_device(0)
claims = bench.cfg2_claims(1234, "cuda")
for s in range(3):
    bench.prove_step_batched([claims], s, zb)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    bench.prove_step_batched([claims], 9, zb)
    torch.cuda.synchronize()
prof.export_chrome_trace(os.path.join(out, "cfg2_step.json"))
ev = json.load(open(os.path.join(out, "cfg2_step.json")))["traceEvents"]
k = sorted((e for e in ev if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")),
           key=lambda e: e["ts"])
t0 = k[0]["ts"]
busy = 0.0
lines = []
prev_end = t0
for e in k:
    gap = e["ts"] - prev_end
    busy += e["dur"]
    lines.append("%9.1f %7.1f gap %7.1f s%-3s %s" % (e["ts"] - t0, e["dur"], gap,
                                                     e["args"].get("stream", "?"), e["name"][:90]))
    prev_end = max(prev_end, e["ts"] + e["dur"])
span = prev_end - t0
lines.append("span %.1f us, kernel-busy %.1f us (%.0f%%), %d ops" % (span, busy, 100 * busy / span,
                                                                  len(k)))
open(os.path.join(out, "cfg2_timeline.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines[-60:]))
