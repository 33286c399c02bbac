timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scratch/trace_cfg2.py; python scratch/trace_cfg2.py
ZKL_NO_PAIR=1 python scratch/trace_cfg2.py
ZKL_TRACE=1 python scratch/trace_cfg2.py 2>&1 | grep "matmul (11,12,12)\|n=11 k=2\|n=12 k=2" | head -6
