# r02: paired rounds in the cluster kernel (PROD2 / SUM2PROD2 over Fr)
O=gpurun_out/r02bw; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matmul or sumcheck or golden or host_tail or zero_u or stepwise" > $O/tests.log 2>&1; echo tests rc=$?; tail -3 $O/tests.log
for la in 1 1 0; do
ZKL_PAIRED=$la timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$la.json 2> $O/bench_$la.err; echo bench la=$la rc=$?
python -c "import json; d=json.loads(open('$O/bench_$la.json').read().strip().splitlines()[-1]); print($la, d['ms_per_step'], d['e2e']['ms_per_step'])"
done
ZKL_TRACE=4 python tools/prof/cfg2_trace.py > $O/trace.log 2>&1
