timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --no-cpu --steps 8 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['cfg3']['ms_per_proof'], d['cfg3']['sumcheck_ms_per_proof'], d['cfg3']['sumcheck_roofline']['achieved'])"
