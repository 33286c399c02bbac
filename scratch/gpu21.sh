timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['eq_tables'], d['round_engine']['us_per_round'], d['roofline']['gpu_ms_per_step'])"
