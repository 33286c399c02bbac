# r02: fully unrolled Montgomery product (ZKL_MUL_UNROLLED) vs rolled: cfg2, cfg3, block
O=gpurun_out/r02af; mkdir -p $O
for v in default unrolled; do
  if [ $v = unrolled ]; then export ZKL_LIB=build/variants/unrolled/libzkl_b200.so; else unset ZKL_LIB; fi
  timeout 1500 python bench.py --steps 10 --warmup 3 --no-cpu --no-cfg5 > $O/bench_$v.json 2> $O/err_$v; echo $v rc=$?
  python -c "import json; d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['cfg3']['ms_per_proof'], d['cfg4']['block_proof_s'], d['cfg4']['verifier_accept'])"
done
