"""GPU timeline (torch.profiler / CUPTI) of one end-to-end cfg2 step as
bench.py times it: layer tensors copied from pinned host memory, witness
products on the device, two batched proofs."""
import itertools
import os
import sys

sys.path[:0] = [".", "tests/golden"]
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2508_21393_b200 as zb  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/e2e_timeline"
os.makedirs(out, exist_ok=True)
torch.cuda.set_device(0)
layer_host = [torch.from_numpy(a).pin_memory() for a in bench.cfg2_host(1234)]
layer_dev = [torch.empty_like(h, device="cuda") for h in layer_host]
X_h, W_h, AL_h, BL_h, dY_h = layer_host
groups = [(X_h, AL_h, BL_h), (W_h,), (dY_h,)]
group_of = {"X": 0, "AL": 0, "BL": 0, "W": 1, "dY": 2}
gbufs = [(layer_dev[0], layer_dev[2], layer_dev[3]), (layer_dev[1],), (layer_dev[4],)]
stager = D.Staged()
prod_bufs, derived, calls = {}, {}, [0]


def igemm_into(a, b):
    key = (calls[0], a.shape[0], b.shape[1])
    calls[0] += 1
    buf = prod_bufs.get(key)
    if buf is None:
        buf = prod_bufs[key] = torch.empty((a.shape[0], b.shape[1]), dtype=torch.int64,
                                           device="cuda")
    return D.igemm16(a.contiguous(), b.contiguous(), out=buf)


def step(seed):
    stager.stage(groups, out=gbufs)
    waited = set()

    def need(name):
        g = group_of.get(name)
        if g is not None and g not in waited:
            stager.ready(g)
            waited.add(g)

    calls[0] = 0
    gen = bench.cfg2_layer_claims(*layer_dev, igemm_into, need=need, keep=derived)
    bench.prove_step_batched([itertools.islice(gen, 2), gen], seed, zb)


for s in range(4):
    step(s)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step(9)
    torch.cuda.synchronize()
prof.export_chrome_trace(os.path.join(out, "e2e_step.json"))
import json  # noqa: E402

ev = json.load(open(os.path.join(out, "e2e_step.json")))["traceEvents"]
k = sorted((e for e in ev if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")),
           key=lambda e: e["ts"])
t0 = k[0]["ts"]
lines, prev_end, busy = [], t0, 0.0
for e in k:
    lines.append("%9.1f %7.1f gap %7.1f s%-3s %s" % (e["ts"] - t0, e["dur"], e["ts"] - prev_end,
                                                     e["args"].get("stream", "?"), e["name"][:90]))
    prev_end = max(prev_end, e["ts"] + e["dur"])
    busy += e["dur"]
lines.append("span %.1f us, busy %.1f us, %d ops" % (prev_end - t0, busy, len(k)))
open(os.path.join(out, "e2e_timeline.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(l for l in lines if "Memcpy" in l or "igemm" in l or "span" in l))
