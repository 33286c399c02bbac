# r02: e2e witness enqueue on a helper thread
O=gpurun_out/r02bo; mkdir -p $O
for i in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$i.json 2> $O/bench_$i.err; echo bench rc=$?
python -c "import json; d=json.loads(open('$O/bench_$i.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'])"
done
ZKL_E2E_SERIAL=1 timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_serial.json 2> $O/bench_serial.err; echo serial rc=$?
python -c "import json; d=json.loads(open('$O/bench_serial.json').read().strip().splitlines()[-1]); print('serial', d['ms_per_step'], d['e2e']['ms_per_step'])"
