set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_v9.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gputest_v9.log
timeout 600 python bench.py > gpurun_out/bench_v9.json 2> gpurun_out/bench_v9.err; echo "bench rc=$?"
cat gpurun_out/bench_v9.json
