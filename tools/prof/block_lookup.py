"""The HBM-bound block passes for ncu: a 2^27-entry rescale witness, its
quant_range histogram (k_range_count16) and lift."""
import sys

sys.path[:0] = ['.']
import torch  # noqa: E402

import bench  # noqa: E402

torch.cuda.cudart().cudaProfilerStart()
bench.run_hbm_kernels(6500.0)
torch.cuda.cudart().cudaProfilerStop()
print("ok")
