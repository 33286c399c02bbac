# r02: host tail length re-check with paired rounds (ZKL_HOST_TAIL 4 / 5 / 6)
O=gpurun_out/r02cc; mkdir -p $O
for h in 4 5 6 4 5 6 4 5 6; do
  ZKL_HOST_TAIL=$h timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$h.json 2> $O/bench_$h.err
  python -c "import json; d=json.loads(open('$O/bench_$h.json').read().strip().splitlines()[-1]); print($h, d['ms_per_step'], d['e2e']['ms_per_step'])"
done
