# r02: int16 tensor-core row matvec tile width / occupancy variants
O=gpurun_out/r02bp; mkdir -p $O
python tools/prof/mv16_time.py > $O/mv16_default.json 2>&1; cat $O/mv16_default.json
for v in t256m2 t128m2 t128m3 t64m4; do
  ZKL_LIB=build/variants/$v/libzkl_b200.so python tools/prof/mv16_time.py > $O/mv16_$v.json 2>&1; cat $O/mv16_$v.json
done
for v in default t128m3 t64m4; do
  if [ $v = default ]; then L=""; else L="ZKL_LIB=build/variants/$v/libzkl_b200.so"; fi
  env $L timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$v.json 2> $O/bench_$v.err
  python -c "import json; d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel_only']['frac'])"
done
