timeout 900 python -m pytest tests -m gpu -x -q -k "matmul or zkmat or stepwise" 2>&1 | tail -2
python scratch/trace_cfg2.py; python scratch/trace_cfg2.py
ZKL_NO_EARLY=1 python scratch/trace_cfg2.py
ZKL_TRACE=1 python scratch/trace_cfg2.py 2>&1 | grep "matmul (11,12,12)" | head -4
