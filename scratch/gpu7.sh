ZKL_TRACE=1 timeout 300 python scratch/trace2.py 2>&1 | grep "zkl trace\] matmul" | sed -n 17,32p
