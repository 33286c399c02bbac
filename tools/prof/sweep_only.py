"""The cfg5 sweep points only (timing / occupancy experiments):
    python tools/prof/sweep_only.py 24 26 28"""
import json
import sys

sys.path[:0] = ['.']
import bench  # noqa: E402

rows = bench.run_sweep([int(a) for a in sys.argv[1:]] or [24, 26, 28], 4.2e10)
print(json.dumps([{k: r[k] for k in ("n", "sumcheck_ms", "mont_products_per_s",
                                     "achieved_gbs", "bit_exact_dense_vs_factored")}
                  for r in rows]))
