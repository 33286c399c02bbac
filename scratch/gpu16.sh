ncu --set full --import-source on --clock-control none -k regex:k_mvf_rows -c 1 -o gpurun_out/mvrows python scratch/mv_bench.py > /dev/null 2>&1; echo rc=$?
ncu --set full --import-source on --clock-control none -k regex:k_mvf_cols -c 1 -o gpurun_out/mvcols python scratch/mv_bench.py > /dev/null 2>&1; echo rc=$?
