python -m pytest tests -m gpu -x -q -k "matvec or matmul" 2>&1 | tail -1
for w in 148 296 592 1184; do echo "--- want $w"; ZKL_MV_WANT=$w python scratch/mv_bench.py; done
