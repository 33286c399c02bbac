mkdir -p gpurun_out/p8
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py > gpurun_out/p8/bench.json 2> gpurun_out/p8/bench.err; tail -1 gpurun_out/p8/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['clocks'], d['cpu_baseline']['value'], d['cfg3']['ms_per_proof'])"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/p8/launches.csv python scratch/prof_step.py > /dev/null 2>&1; echo ncu1 rc=$?
python tools/ncu_launches.py gpurun_out/p8/launches.csv > gpurun_out/p8/launches.summary.txt; head -14 gpurun_out/p8/launches.summary.txt
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_mvw_rows -c 1 -o gpurun_out/p8/k_mvw_rows python scratch/prof_step.py > /dev/null 2>&1; echo ncu2 rc=$?
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_mvf_cols -c 1 -o gpurun_out/p8/k_mvf_cols python scratch/prof_step.py > /dev/null 2>&1; echo ncu3 rc=$?
python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/p8/bench_reference.json; cat gpurun_out/p8/bench_reference.json | cut -c1-300
