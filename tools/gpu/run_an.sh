# r02: four-lane eq tree
O=gpurun_out/r02an; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py tests/test_gpu_block.py tests/test_gpu_shard.py -q -x > $O/tests.log 2>&1; echo tests rc=$?; tail -3 $O/tests.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench.json 2> $O/bench.err; echo bench rc=$?; tail -3 $O/bench.err

for f in $O/bench.json $O/bench_nographs.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['e2e']['ms_per_step'], d['gpu_launches'], d['roofline']['measured_over'][-80:])"; done
