"""int64 matrix x Fr vector products (the zkMat C matvecs) on cfg2's largest
shape, rows and columns: per-call time and GB/s.  Run once with the default
(wide-accumulator) kernels and once with ZKL_MATVEC_FAST64=1 (16-bit chunks
on mad.wide)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_21393_b200 import _native as N  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402

spec = D.FR
rows, cols = 2048, 4096
g = torch.Generator(device="cuda").manual_seed(5)
M = torch.randint(-(1 << 42), 1 << 42, (rows, cols), device="cuda", generator=g, dtype=torch.int64)
out = {"variant": "wide-accumulator" if os.environ.get("ZKL_MV_TC64") == "0" else "tensor cores"}
for tr, n_in, n_out in ((0, cols, rows), (1, rows, cols)):
    x = D.upload([(i * 7919 + 13) ** 5 for i in range(n_in)], spec)
    y = D.empty(spec, n_out)

    def call():
        N.check(N.lib().zkl_matvec(spec.fid, N.MT_I64, D.ptr(M), rows, cols, tr, D.ptr(x),
                                   D.ptr(y), D.stream()))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        call()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    out["cols" if tr else "rows"] = {"us": ms * 1e3, "gbs": rows * cols * 8 / ms / 1e6,
                                     "checksum": D.download(y, spec, 4)[0] % 1000003}
print(json.dumps(out))
