mkdir -p gpurun_out/v27
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v27/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/v27/gpu_tests.log
python scratch/lookup_prof.py 27 2>&1 | tail -20
timeout 600 python scratch/block_prof.py stages > gpurun_out/v27/block_prof.log 2>&1; echo "rc=$?"; head -1 gpurun_out/v27/block_prof.log; grep -A16 -- "--- stages" gpurun_out/v27/block_prof.log
