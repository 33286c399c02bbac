# r02: e2e with witness stream + reordered claims; host profile of a step
O=gpurun_out/r02q; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench.json 2> $O/bench.err; echo bench rc=$?; tail -5 $O/bench.err
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], json.dumps(d['e2e']))"
timeout 600 python tools/prof/cfg2_pyprof.py > $O/pyprof.txt 2>&1; head -50 $O/pyprof.txt
