# r02: timed pass without profiler brackets, profiled second pass; e2e warm-up
O=gpurun_out/r02z; mkdir -p $O
for i in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_prof$i.json 2> $O/err1

done
for f in $O/bench_prof1.json $O/bench_prof2.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['operands_copied']['ms_per_step'], d['roofline']['frac'], d['roofline']['measured_over'])"; done
