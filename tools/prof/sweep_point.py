"""One cfg5 sweep point (the reference's replicated zkMat claim on the dense
fused round/fold engine) for ncu.  With ZKL_PROFILE_REPLAY=1 the proof runs
stepwise and the production kernels (k_sumcheck_persistent<EvZkMat> ->
k_sumcheck_cluster) then replay it on recorded challenges:

  ZKL_PROFILE_REPLAY=1 ncu --set full -k regex:"k_sumcheck_(persistent|cluster)" \
      -c 2 python tools/prof/sweep_point.py 26
"""
import sys

sys.path[:0] = ['.', 'tests/golden']
import torch  # noqa: E402

import bench  # noqa: E402

torch.cuda.cudart().cudaProfilerStart()
bench.run_sweep([int(sys.argv[1]) if len(sys.argv) > 1 else 26])
torch.cuda.cudart().cudaProfilerStop()
print("ok")
