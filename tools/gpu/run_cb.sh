# r02: pause between a polling warp's reads of host memory (ZKL_POLL_SLEEP_NS variants)
O=gpurun_out/r02cb; mkdir -p $O
for v in default sl200 sl500 default sl200 sl500; do
  if [ $v = default ]; then L=""; else L="ZKL_LIB=build/variants/$v/libzkl_b200.so"; fi
  env $L timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$v.json 2> $O/bench_$v.err
  python -c "import json; d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
