# r02: ADX host Montgomery product + 3-product host tail; lane passes default 4
O=gpurun_out/r02bc; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matmul or sumcheck or golden or host_tail or logup" > $O/tests.log 2>&1; echo tests rc=$?; tail -1 $O/tests.log
for i in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$i.json 2> $O/bench_$i.err; echo bench rc=$?
python -c "import json; d=json.loads(open('$O/bench_$i.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'])"
done
ZKL_TRACE=2 python tools/prof/cfg2_trace.py > $O/trace.log 2>&1
