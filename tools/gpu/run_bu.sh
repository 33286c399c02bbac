# r02: paired-round pass threshold sweep (ZKL_PAIR_PASSES)
O=gpurun_out/r02bu; mkdir -p $O
for p in 1 2 4 1 2 4; do
  ZKL_PAIR_PASSES=$p timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$p.json 2> $O/bench_$p.err
  python -c "import json; d=json.loads(open('$O/bench_$p.json').read().strip().splitlines()[-1]); print($p, d['ms_per_step'], d['e2e']['ms_per_step'])"
done
