# r02: cp.async-pipelined int64 TC matvecs
O=gpurun_out/r02x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matvec or matmul or cfg2" > $O/tests.log 2>&1; echo tests rc=$?; tail -3 $O/tests.log
python tools/prof/mv64_time.py > $O/mv64.jsonl 2>&1; ZKL_MV_TC64=0 python tools/prof/mv64_time.py >> $O/mv64.jsonl 2>&1; cat $O/mv64.jsonl
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench.json 2> $O/bench.err; echo bench rc=$?; tail -3 $O/bench.err
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'])"
