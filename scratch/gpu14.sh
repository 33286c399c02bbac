python -m pytest tests -m gpu -x -q -k "matvec or matmul" 2>&1 | tail -1
for w in 592 1184 2368; do echo "--- warps $w"; ZKL_MV_WARPS=$w python scratch/mv_bench.py; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mv_launch.csv python scratch/mv_bench.py > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/mv_launch.csv | head -12
