mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "lookup or multiplicities or pair" > gpurun_out/t11.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t11.log
grep -n "Error\|error" gpurun_out/t11.log | head
timeout 300 python scratch/cfg3.py
