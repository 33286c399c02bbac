mkdir -p gpurun_out/v28
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v28/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/v28/gpu_tests.log
timeout 600 python scratch/block_prof.py > gpurun_out/v28/block_prof.log 2>&1; echo "rc=$?"; head -1 gpurun_out/v28/block_prof.log; grep -A16 -- "--- by" gpurun_out/v28/block_prof.log
timeout 600 python scratch/block_run.py 13b 2 2>&1 | grep "block "
