python scratch/mv_bench.py
echo "--- slow"
ZKL_MATVEC_SLOW=1 python scratch/mv_bench.py
ncu --set full --import-source on --clock-control none -k regex:k_mvf -c 2 -o gpurun_out/mvf_full python scratch/mv_bench.py > gpurun_out/ncu_mvf.log 2>&1; echo ncu rc=$?
