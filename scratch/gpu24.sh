ZKL_MATVEC_FAST=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mvf.csv python scratch/mv_bench.py > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/mvf.csv | head -12
echo ---slow
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mvs.csv python scratch/mv_bench.py > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/mvs.csv | head -8
