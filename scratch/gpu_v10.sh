mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "lookup or multiplicities or pair" > gpurun_out/t10.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t10.log
timeout 300 python scratch/cfg3.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg3_launch10.csv python scratch/cfg3.py 25 > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_launches.py gpurun_out/cfg3_launch10.csv | head -30
