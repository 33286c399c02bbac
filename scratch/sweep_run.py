import json, sys
sys.path[:0] = ['.', 'tests/golden']
import torch, bench
ns = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [20, 22, 24, 26, 28, 30]
bench.run_sweep([20])  # warm-up (lazy module load)
for r in bench.run_sweep(ns, 4.2e10):
    print(json.dumps(r), flush=True)
print("peak mem %.1f GB" % (torch.cuda.max_memory_allocated() / 1e9))
