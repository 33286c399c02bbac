# r02: replay-mode fix check, lift/histogram tests, ncu of the production dense kernels
set -x
O=gpurun_out/r02e; mkdir -p $O
ZKL_PROFILE_REPLAY=1 timeout 600 python tools/prof/replay_dbg.py > $O/replay_dbg.log 2>&1; echo replay rc=$?; tail -8 $O/replay_dbg.log
timeout 1200 python -m pytest tests/test_gpu_nonlinear.py tests/test_gpu_parity.py -q -rf -k "lift or range or replay or stepwise" > $O/tests.log 2>&1; echo tests rc=$?; tail -5 $O/tests.log
timeout 900 env ZKL_PROFILE_REPLAY=1 ncu --set full --import-source on --clock-control none -k regex:"k_sumcheck_(persistent|cluster)" -c 2 -o $O/dense26_full python tools/prof/sweep_point.py 26 > $O/ncu_dense.log 2>&1; echo ncu_dense rc=$?; tail -3 $O/ncu_dense.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lift16 -c 1 -o $O/hbm_k_lift16_direct python tools/prof/block_lookup.py > $O/ncu_lift.log 2>&1; echo ncu lift rc=$?
python bench.py --steps 3 --warmup 3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_hbm.json 2>$O/bench_hbm.err; echo bench rc=$?; python -c "import json; d=json.loads(open('$O/bench_hbm.json').read().strip().splitlines()[-1]); print({k: (round(v['ms'],3), round(v['frac'],3)) for k,v in d['hbm_kernels']['kernels'].items()}, d['cfg3']['ms_per_proof'])"
