import sys
sys.path[:0] = ['.', 'tests/golden']
import torch, bench
torch.cuda.cudart().cudaProfilerStart()
bench.run_sweep([int(sys.argv[1]) if len(sys.argv) > 1 else 26])
torch.cuda.cudart().cudaProfilerStop()
print("ok")
