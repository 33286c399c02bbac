# r02: cost of the profiler brackets in the timed region
O=gpurun_out/r02y; mkdir -p $O
for i in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_prof$i.json 2> $O/err1
ZKL_BENCH_NOPROF=1 timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_noprof$i.json 2> $O/err2
done
for f in $O/bench_prof1.json $O/bench_noprof1.json $O/bench_prof2.json $O/bench_noprof2.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['e2e']['ms_per_step'])"; done
