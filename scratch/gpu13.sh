python -m pytest tests -m gpu -x -q -k "matvec or matmul" 2>&1 | tail -1
for w in 1184 2368 3552 4736; do echo "--- warps $w"; ZKL_MV_WARPS=$w python scratch/mv_bench.py; done
