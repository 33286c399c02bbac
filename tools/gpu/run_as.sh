# r02: e2e with the second batch's products on a witness stream under the first batch
O=gpurun_out/r02as; mkdir -p $O
for v in overlap serial; do
  if [ $v = serial ]; then export ZKL_E2E_SERIAL=1; else unset ZKL_E2E_SERIAL; fi
  timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$v.json 2> $O/err_$v; echo $v rc=$?; tail -2 $O/err_$v
  python -c "import json; d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
