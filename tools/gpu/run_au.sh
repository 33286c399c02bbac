# r02: barrier-free matvec finish kernels
O=gpurun_out/r02au; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matvec or matmul or cfg2" > $O/tests.log 2>&1; echo tests rc=$?; tail -1 $O/tests.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench.json 2> $O/bench.err; echo bench rc=$?
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel_only']['frac'])"
