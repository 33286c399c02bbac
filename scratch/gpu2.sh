mkdir -p gpurun_out
ZKL_TRACE=1 timeout 300 python scratch/trace_step.py > gpurun_out/trace.log 2>&1; echo "trace rc=$?"
grep -v "zkl trace" gpurun_out/trace.log | tail -12
grep "zkl trace" gpurun_out/trace.log | tail -24
ZKL_NO_PERSISTENT=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python scratch/prof_step.py > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python scratch/launches.py gpurun_out/launches.csv > gpurun_out/launches.summary.txt 2>&1
head -30 gpurun_out/launches.summary.txt
ZKL_NO_PERSISTENT=1 timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_mv_rows -c 1 -o gpurun_out/mv_rows_full python scratch/prof_step.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
