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
import test_gpu_parity_scale as S
for name, fn in [("cfg5-24", S.test_cfg5_dense_replicated_claim_matches_oracle),
                 ("prod3-16", lambda: T.test_sumcheck_shapes_vs_oracle('test', 16, 'prod3')),
                 ("s2p2-15", lambda: T.test_sumcheck_shapes_vs_oracle('big', 15, 'sum2prod2'))]:
    try:
        fn(); print(name, "ok", flush=True)
    except Exception as e:
        print(name, "FAIL", str(e)[:300], flush=True)
