# r02: cluster lane-mode passes sweep (ZKL_CLUSTER_LANE_PASSES) on cfg2 + per-round trace
O=gpurun_out/r02ba; mkdir -p $O
for p in 1 2 4 8; do
  ZKL_CLUSTER_LANE_PASSES=$p timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$p.json 2> $O/bench_$p.err; echo bench p=$p rc=$?
  python -c "import json; d=json.loads(open('$O/bench_$p.json').read().strip().splitlines()[-1]); print($p, d['ms_per_step'], d['e2e']['ms_per_step'])"
done
ZKL_TRACE=2 ZKL_CLUSTER_LANE_PASSES=4 python tools/prof/cfg2_trace.py > $O/trace4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matmul or sumcheck or golden or host_tail" > $O/tests.log 2>&1; echo tests rc=$?; tail -1 $O/tests.log
