# r02: host tail rounds for the zkMat W / V phases (ZKL_HOST_TAIL sweep)
O=gpurun_out/r02av; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matvec or matmul or cfg2 or golden or sumcheck" > $O/tests.log 2>&1; echo tests rc=$?; tail -1 $O/tests.log
for h in 0 3 4 5 6; do
  ZKL_HOST_TAIL=$h timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$h.json 2> $O/bench_$h.err; echo bench h=$h rc=$?
  python -c "import json; d=json.loads(open('$O/bench_$h.json').read().strip().splitlines()[-1]); print($h, d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel_only']['frac'])"
done
