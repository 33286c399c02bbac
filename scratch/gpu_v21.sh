mkdir -p gpurun_out/v21
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v21/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/v21/gpu_tests.log
timeout 600 python bench.py > gpurun_out/v21/bench.json 2> gpurun_out/v21/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/v21/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'], d['cfg3']['ms_per_proof'], d['cfg3']['sumcheck_ms_per_proof'], d['roofline']['frac'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/v21/bench_reference.json 2>&1; tail -1 gpurun_out/v21/bench_reference.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/v21/launches.csv python scratch/prof_step.py > /dev/null 2>&1; echo ncu1 rc=$?
python tools/ncu_launches.py gpurun_out/v21/launches.csv > gpurun_out/v21/launches.summary.txt; head -14 gpurun_out/v21/launches.summary.txt
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_round -c 2 -o gpurun_out/v21/k_round python scratch/prof_step.py > /dev/null 2>&1; echo ncu2 rc=$?
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_mvw_rows -c 1 -o gpurun_out/v21/k_mvw_rows python scratch/prof_step.py > /dev/null 2>&1; echo ncu3 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v21/cfg3_launches.csv python scratch/cfg3.py 25 > /dev/null 2>&1; echo ncu4 rc=$?
python tools/ncu_launches.py gpurun_out/v21/cfg3_launches.csv > gpurun_out/v21/cfg3_launches.summary.txt; head -12 gpurun_out/v21/cfg3_launches.summary.txt
