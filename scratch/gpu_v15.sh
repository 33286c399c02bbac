timeout 600 python -m pytest tests -m gpu -x -q -k "lookup" 2>&1 | tail -1
ZKL_TRACE=1 python scratch/cfg3_prof.py 2>&1 | grep "zkl trace" | head -2
python scratch/cfg3_prof.py 2>&1 | head -4
