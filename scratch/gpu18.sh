mkdir -p gpurun_out/p7
python bench.py 2>gpurun_out/p7/bench.err | tail -1 > gpurun_out/p7/bench.json; python -c "import json; d=json.load(open('gpurun_out/p7/bench.json')); print(d['ms_per_step'], d['value'], d['clocks'], d['round_engine']['us_per_round'], d['roofline']['achieved'])"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/p7/launches.csv python scratch/prof_step.py > /dev/null 2>&1; echo ncu1 rc=$?
python tools/ncu_launches.py gpurun_out/p7/launches.csv > gpurun_out/p7/launches.summary.txt; head -12 gpurun_out/p7/launches.summary.txt
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_mv_rows -c 1 -o gpurun_out/p7/k_mv_rows python scratch/prof_step.py > /dev/null 2>&1; echo ncu2 rc=$?
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_mv_cols -c 1 -o gpurun_out/p7/k_mv_cols python scratch/prof_step.py > /dev/null 2>&1; echo ncu3 rc=$?
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_round -c 1 -o gpurun_out/p7/k_round python scratch/prof_step.py > /dev/null 2>&1; echo ncu4 rc=$?
