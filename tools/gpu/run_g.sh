# r02: dense-engine occupancy experiment (255 vs 128 registers), matvec prefetch check,
# ncu of the dense EvZkMat production kernels
set -x
O=gpurun_out/r02g; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -q -x -k "matvec or matmul or cfg2" > $O/mv_tests.log 2>&1; echo mvtests rc=$?; tail -2 $O/mv_tests.log
for v in default minb2; do
  if [ $v = default ]; then L=""; else L="ZKL_LIB=build/variants/$v/libzkl_b200.so"; fi
  env $L timeout 900 python tools/prof/sweep_only.py 24 26 28 > $O/sweep_$v.json 2>&1; echo sweep $v rc=$?; tail -1 $O/sweep_$v.json
  env $L timeout 900 python bench.py --steps 10 --warmup 3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$v.json 2> $O/bench_$v.err; echo bench $v rc=$?
  python -c "import json; d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['frac'], d['roofline']['gpu_ms_per_step'], d['cfg3']['ms_per_proof'], d['round_engine']['us_per_round'])"
done
timeout 900 env ZKL_PROFILE_REPLAY=1 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"EvZkMat" -c 2 -o $O/dense26_zkmat python tools/prof/sweep_point.py 26 > $O/ncu_dense.log 2>&1; echo ncu_dense rc=$?; tail -2 $O/ncu_dense.log
