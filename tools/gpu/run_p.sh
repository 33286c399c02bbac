# r02: e2e from layer tensors (device witness) vs operands copied
O=gpurun_out/r02p; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench.json 2> $O/bench.err; echo bench rc=$?; tail -5 $O/bench.err
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], json.dumps(d['e2e']))"
