import sys
sys.path[:0] = ['.', 'tests/golden']
import json, bench
print(json.dumps(bench.run_hbm_kernels(6549.1), indent=1))
