mkdir -p gpurun_out/v40
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v40/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/v40/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/v40/bench.json 2> gpurun_out/v40/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/v40/bench.err
tail -1 gpurun_out/v40/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['gpu_ms_per_step'], d['cfg3']['ms_per_proof'], d['lora_block_proof_s'], d['cfg5']['block_13b']['block_proof_s'], d['clocks'], {k: round(v['frac'],2) for k, v in d['hbm_kernels']['kernels'].items()})"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/v40/bench_reference.json 2>&1; tail -1 gpurun_out/v40/bench_reference.json | cut -c1-150
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/v40/launches.csv python scratch/prof_step.py > /dev/null 2>&1; echo ncu1 rc=$?
python tools/ncu_launches.py gpurun_out/v40/launches.csv > gpurun_out/v40/launches.summary.txt; head -12 gpurun_out/v40/launches.summary.txt
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_mvt_rows|k_mvt_cols" -c 2 -o gpurun_out/v40/matvec_full python scratch/prof_step.py > /dev/null 2>&1; echo ncu2 rc=$?
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
