ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg3_launch.csv python scratch/cfg3.py 25 > /dev/null 2>&1; echo rc=$?
python tools/ncu_launches.py gpurun_out/cfg3_launch.csv | head -24
