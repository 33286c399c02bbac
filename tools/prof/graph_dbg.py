"""Graph-cached zkMat phase inputs vs the eager path on the golden matmul
cases: the same claim proven repeatedly (eager, capture, replays)."""
import sys

sys.path[:0] = [".", "tests", "tests/golden"]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import FIELDS, load_golden  # noqa: E402
import paper_2508_21393_b200 as zb  # noqa: E402
from paper_2508_21393_b200.gadgets import DeviceMatrix  # noqa: E402
from paper_2508_21393_b200.transcript import Transcript  # noqa: E402
import test_gpu_parity as T  # noqa: E402

for ci, c in enumerate(load_golden("matmul.json")):
    p = FIELDS[c["field"]]
    a, b, cm = T._mm_data(c)
    dims = tuple(c["dims"])
    for dt in (torch.int16, torch.int64):
        if dt == torch.int16 and (np.abs(a).max() > 32767 or np.abs(b).max() > 32767):
            continue
        A, B = T._dev(a, dt), T._dev(b, dt)
        C = T._dev(cm, torch.int64)
        res = []
        for it in range(4):
            t = Transcript.from_state(bytes.fromhex(c["state_before"]), p)
            rounds, point, finals = zb.matmul_sumcheck(A, B, C, dims, t)
            res.append(([list(r) for r in rounds] == c["rounds"], list(finals) == c["final_values"]))
        print(ci, c["field"], dims, dt, res, flush=True)
