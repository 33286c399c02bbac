timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mvf.csv python scratch/mv_bench.py > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/mvf.csv | head -8
python bench.py --no-cpu --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['gpu_ms_per_step'], d['roofline']['achieved'], d['round_engine']['us_per_round'], d['cfg3']['ms_per_proof'])"
