timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
mkdir -p gpurun_out/p7
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/p7/launches.csv python scratch/prof_step.py > /dev/null 2>&1; echo ncu1 rc=$?
python tools/ncu_launches.py gpurun_out/p7/launches.csv > gpurun_out/p7/launches.summary.txt; head -14 gpurun_out/p7/launches.summary.txt
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_round -c 1 -o gpurun_out/p7/k_round python scratch/prof_step.py > /dev/null 2>&1; echo ncu4 rc=$?
