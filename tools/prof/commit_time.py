"""GPU Hyrax row commitments: seconds per table and per entry, for random
field tables and for int16-valued ones (the block's tensors), beside the
reference's per-entry cost (46 us, profiles/r02 bench cpu_baseline)."""
import json
import random
import sys
import time
from collections import namedtuple

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2508_21393_b200 import commit_gpu  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402

P = D.MODULUS
Group = namedtuple("Group", "q order cofactor")
Key = namedtuple("Key", "group generators blinding_generator seed max_vars")
grp = Group(96 * P + 1, P, 96)
rnd = random.Random(1)
width = 1 << 12
gens = tuple(pow(rnd.randrange(2, grp.q - 1), 96, grp.q) for _ in range(width))
key = Key(grp, gens, pow(7, 96, grp.q), b"timing", 24)
spec = D.spec_for(P)
t0 = time.perf_counter()
commit_gpu.key_tables(key)
torch.cuda.synchronize()
print(json.dumps({"key_tables_s": time.perf_counter() - t0, "generators": width + 1}))
for n in (16, 20, 22, 24):
    for kind in ("random", "int16"):
        g = torch.Generator(device="cuda").manual_seed(n)
        if kind == "int16":
            x = torch.randint(-32768, 32768, (1 << n,), device="cuda", dtype=torch.int32,
                              generator=g).to(torch.int16)
            dv = D.DeviceVector(D.lift(x, spec), 1 << n, spec)
        else:
            vals = [rnd.randrange(P) for _ in range(1 << min(n, 16))]
            reps = (1 << n) // len(vals)
            dv = D.DeviceVector(D.upload(vals * reps, spec), 1 << n, spec)
        commit_gpu.commit_rows(key, dv, n)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        commit_gpu.commit_rows(key, dv, n)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"num_vars": n, "values": kind, "seconds": dt,
                          "us_per_entry": dt / (1 << n) * 1e6,
                          "speedup_vs_reference_46us": 46e-6 * (1 << n) / dt}), flush=True)
