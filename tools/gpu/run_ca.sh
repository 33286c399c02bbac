# r02: staggered multi-warp challenge polling in the cluster kernel (ZKL_POLL_WARPS)
O=gpurun_out/r02ca; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matmul or sumcheck or golden or host_tail or zero_u or stepwise or logup" > $O/tests.log 2>&1; echo tests rc=$?; tail -1 $O/tests.log
for w in 4 1 4 1 2; do
  ZKL_POLL_WARPS=$w timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err
  python -c "import json; d=json.loads(open('$O/bench_$w.json').read().strip().splitlines()[-1]); print($w, d['ms_per_step'], d['e2e']['ms_per_step'])"
done
