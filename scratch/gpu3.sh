mkdir -p gpurun_out
lscpu | grep -i "model name\|^CPU(s)\|MHz" | head -4
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests.log
ZKL_TRACE=1 timeout 300 python scratch/trace_step.py > gpurun_out/trace.log 2>&1; echo "trace rc=$?"
tail -8 gpurun_out/trace.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench.log
