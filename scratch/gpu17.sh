timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench.json; cat gpurun_out/bench.json | python -m json.tool | head -80
ZKL_MATVEC_FAST=1 timeout 300 python scratch/trace2.py 2>&1 | grep "native=True"
timeout 300 python scratch/trace2.py 2>&1 | grep "native=True"
