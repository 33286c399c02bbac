# r02: batched zkMat driver: parity tests, cfg2 bench, timeline
O=gpurun_out/r02s; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matmul or cfg2 or stepwise" > $O/tests.log 2>&1; echo tests rc=$?; tail -3 $O/tests.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench.json 2> $O/bench.err; echo bench rc=$?; tail -5 $O/bench.err
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['operands_copied']['ms_per_step'], d['round_engine']['us_per_round'])"
