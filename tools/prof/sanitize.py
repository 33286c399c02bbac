"""Small proofs through every production kernel family, for
compute-sanitizer (memcheck / racecheck / synccheck):

    ZKL_FORCE_PERSISTENT=1 compute-sanitizer --tool memcheck python tools/prof/sanitize.py

ZKL_FORCE_PERSISTENT keeps the persistent / cluster round engine under the
sanitizer (it serialises but does not replay kernels, so the host still
answers each round).  Every proof is also checked against the oracle."""
import sys

sys.path[:0] = [".", "tests", "tests/golden"]
import pytest  # noqa: E402
import torch  # noqa: E402

import test_gpu_parity as T  # noqa: E402

torch.cuda.set_device(0)
checks = [
    ("sumcheck prod2 n=10", lambda: T.test_sumcheck_shapes_vs_oracle("big", 6, "prod2")),
    ("sumcheck prod3 n=15 (grid -> cluster)",
     lambda: T.test_sumcheck_shapes_vs_oracle("big", 15, "prod3")),
    ("sumcheck sum2prod2", lambda: T.test_sumcheck_shapes_vs_oracle("test", 16, "sum2prod2")),
    ("sumcheck logup 7 tables", lambda: T.test_sumcheck_random_vs_oracle("big", 7, 3, 10)),
    ("zkMat factored (5,9,3)", lambda: T.test_matmul_factored_vs_oracle("big", (5, 9, 3), "i16",
                                                                         "native")),
    ("zkMat factored int64 (4,6,5)",
     lambda: T.test_matmul_factored_vs_oracle("big", (4, 6, 5), "i64", "native")),
    ("batch inverse", lambda: T.test_batch_inverse_sizes("big", 4097)),
    ("eq table 2-level", lambda: T.test_eq_table_large_two_level("big")),
    ("logUp tiled + indexed (d=2^12, n=2^6)",
     lambda: T.test_lookup_indexed_matches_plain("big", 1 << 12, 1 << 6, pytest.MonkeyPatch())),
]
for name, fn in checks:
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)
import test_gpu_nonlinear as NLT  # noqa: E402

NLT.test_lift_int16_exhaustive("big")
print("ok lift", flush=True)
print("sanitize run complete")
