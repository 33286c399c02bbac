timeout 300 python scratch/trace2.py 2>&1 | tail -30
ZKL_TRACE=1 timeout 300 python scratch/trace2.py 2>&1 | grep "zkl trace" | head -30
