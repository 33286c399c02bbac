mkdir -p gpurun_out/v22
timeout 600 python -m pytest tests/test_gpu_nonlinear.py tests/test_gpu_block.py -x -q > gpurun_out/v22/tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/v22/tests.log
timeout 900 python scratch/block_run.py 7b 2 > gpurun_out/v22/block7b.log 2>&1; echo "block rc=$?"; tail -8 gpurun_out/v22/block7b.log | cut -c1-1500
