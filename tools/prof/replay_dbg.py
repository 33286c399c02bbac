import sys, os
sys.path[:0] = ['.', 'tests', 'tests/golden']
import test_gpu_parity as T
for name, fn in [("s2p2", lambda: T.test_sumcheck_shapes_vs_oracle('big', 6, 'sum2prod2')),
                 ("prod3", lambda: T.test_sumcheck_shapes_vs_oracle('test', 16, 'prod3')),
                 ("rand", lambda: T.test_sumcheck_random_vs_oracle('big', 7, 3, 12)),
                 ("mm", lambda: T.test_matmul_factored_vs_oracle('big', (5, 9, 3), 'i16', 'native'))]:
    try:
        fn(); print(name, "ok", flush=True)
    except Exception as e:
        print(name, "FAIL", str(e)[:300], flush=True)
