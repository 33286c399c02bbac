"""int16 matrix x Fr vector products (the zkMat A / B matvecs) on cfg2's
shapes, rows and columns: per-call time (back to back, with the finish
kernel) and GB/s of the matrix bytes, plus a checksum to compare builds
(ZKL_LIB variants, tools/prof/build_variant.py)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_21393_b200 import _native as N  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402

spec = D.FR
out = {"lib": os.environ.get("ZKL_LIB", "default")}
g = torch.Generator(device="cuda").manual_seed(5)
for rows, cols in ((2048, 4096), (4096, 4096), (4096, 2048)):
    M = torch.randint(-32768, 32768, (rows, cols), device="cuda", generator=g, dtype=torch.int16)
    for tr, n_in, n_out in ((0, cols, rows), (1, rows, cols)):
        x = D.upload([(i * 7919 + 13) ** 5 for i in range(n_in)], spec)
        y = D.empty(spec, n_out)

        def call():
            N.check(N.lib().zkl_matvec(spec.fid, N.MT_I16, D.ptr(M), rows, cols, tr, D.ptr(x),
                                       D.ptr(y), D.stream()))
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50):
            call()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 50
        out["%dx%d %s" % (rows, cols, "cols" if tr else "rows")] = {
            "us": round(ms * 1e3, 2), "gbs": round(rows * cols * 2 / ms / 1e6, 1),
            "checksum": D.download(y, spec, 4)[0] % 1000003}
print(json.dumps(out))
