# r02: kernel-only (CUPTI) matvec roofline in the bench line
O=gpurun_out/r02al; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench.json 2> $O/bench.err; echo bench rc=$?; tail -3 $O/bench.err
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); r=d['roofline']; print(d['ms_per_step'], r['frac'], json.dumps(r['kernel_only']))"
