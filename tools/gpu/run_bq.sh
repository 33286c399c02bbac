# r02: V inputs split at the W host tail (Z = E_hi^T B under the tail)
O=gpurun_out/r02bq; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -q -x -k "matmul or host_tail or zero_u or stepwise or cfg2 or graph" > $O/tests.log 2>&1; echo tests rc=$?; tail -2 $O/tests.log
for i in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$i.json 2> $O/bench_$i.err; echo bench rc=$?
python -c "import json; d=json.loads(open('$O/bench_$i.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'])"
done
