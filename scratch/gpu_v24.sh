mkdir -p gpurun_out/v24
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v24/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/v24/gpu_tests.log
timeout 900 python scratch/sweep_run.py 20,22,24,26,28,30 > gpurun_out/v24/sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/v24/sweep.log | cut -c1-400
timeout 900 python scratch/block_run.py 13b 2 > gpurun_out/v24/block13b.log 2>&1; echo "block13 rc=$?"; grep -E "block|setup" gpurun_out/v24/block13b.log | cut -c1-300; tail -3 gpurun_out/v24/block13b.log | cut -c1-1500
