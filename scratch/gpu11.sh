python -m pytest tests -m gpu -x -q -k "matvec or matmul" 2>&1 | tail -1
ncu --set full --import-source on --clock-control none -k regex:k_mvf -c 2 -o gpurun_out/mvf2 python scratch/mv_bench.py > gpurun_out/ncu_mvf2.log 2>&1; echo ncu rc=$?
