"""Time the exact int16 GEMM (zkl_igemm_i16) against the float64 cuBLAS GEMM on
the LoRA block's witness shapes (Llama-7B, seq 2048)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_21393_b200 import device as D  # noqa: E402

SHAPES = [(2048, 4096, 4096), (2048, 4096, 16), (16, 2048, 4096), (2048, 4096, 11008), (4096, 2048, 4096),
          (2048, 128, 2048), (2048, 2048, 128), (4096, 2048, 11008)]


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


out = []
for M, K, N in SHAPES:
    a = torch.randint(-2 ** 15, 2 ** 15, (M, K), device="cuda", dtype=torch.int32).to(torch.int16)
    b = torch.randint(-2 ** 15, 2 ** 15, (K, N), device="cuda", dtype=torch.int32).to(torch.int16)
    ti = t(lambda: D.igemm16(a, b))
    ad, bd = a.double(), b.double()
    tf = t(lambda: torch.matmul(ad, bd))
    tfc = t(lambda: torch.matmul(a.double(), b.double()).round_().long())
    macs = M * K * N
    out.append(dict(shape=[M, K, N], igemm_ms=ti, fp64_ms=tf, fp64_with_casts_ms=tfc,
                    igemm_tops_int8=4 * macs * 2 / ti / 1e9, fp64_tflops=2 * macs / tf / 1e9))
    print(json.dumps(out[-1]), flush=True)
