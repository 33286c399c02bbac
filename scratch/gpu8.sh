timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python scratch/trace2.py 2>&1 | grep "native=True"
ZKL_TRACE=1 timeout 300 python scratch/trace2.py 2>&1 | grep "zkl trace" | sed -n 33,44p
