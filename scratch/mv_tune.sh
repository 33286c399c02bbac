mkdir -p gpurun_out/mvt
for cfg in "2 2 1" "2 4 1" "2 2 2" "4 2 1"; do
  set -- $cfg
  ZKL_MVW_RW=$1 ZKL_MVW_WAVES=$2 ZKL_MVW_GROUPS=$3 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread --clock-control none -k regex:k_mvw_rows --csv --log-file gpurun_out/mvt/rw$1_w$2_g$3.csv python scratch/mv_bench.py > /dev/null 2>&1
done
