"""Witness-pass breakdown: the block witness (prove_block through a
WitnessRecorder) run twice per shape, with the time spent in the int16
tensor-core GEMM accumulated from CUDA events around each call."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2508_21393_b200 import block as BK  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402

P_BIG = D.MODULUS
tables = BK.block_tables(D.spec_for(P_BIG))
acc = {"ms": 0.0, "calls": 0, "shapes": {}}
orig = D.igemm16


def timed_igemm(a, b):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    c = orig(a, b)
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e)
    acc["ms"] += ms
    acc["calls"] += 1
    key = "x".join(map(str, (a.shape[0], a.shape[1], b.shape[1])))
    acc["shapes"][key] = acc["shapes"].get(key, 0.0) + ms
    return c


BK.igemm16 = timed_igemm
for name in sys.argv[1:] or ["7b", "13b"]:
    shape = {"7b": BK.LLAMA2_7B, "13b": BK.LLAMA2_13B}[name]
    w = BK.BlockWitness(shape, seed=1)
    for it in range(2):
        acc.update(ms=0.0, calls=0, shapes={})
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        BK.prove_block(w, BK.WitnessRecorder(tables))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        top = sorted(acc["shapes"].items(), key=lambda kv: -kv[1])[:6]
        print(json.dumps(dict(shape=name, iteration=it, witness_s=dt, igemm_ms=acc["ms"],
                              igemm_calls=acc["calls"], top_shapes=top)), flush=True)
    del w
    torch.cuda.empty_cache()
