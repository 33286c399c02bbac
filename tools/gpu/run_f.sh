# r02: ncu of the production round kernels (recorded-challenge replay) and the cfg2 matvecs,
# an N=2 smoke of bench.py's multi-rank path on this 1-GPU box, the full GPU suite
set -x
O=gpurun_out/r02f; mkdir -p $O
timeout 900 env ZKL_PROFILE_REPLAY=1 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_sumcheck_(persistent|cluster)<Fr255, 4, EvZkMat" -c 2 -o $O/dense26_zkmat python tools/prof/sweep_point.py 26 > $O/ncu_dense.log 2>&1; echo ncu_dense rc=$?; tail -2 $O/ncu_dense.log
timeout 900 env ZKL_PROFILE_REPLAY=1 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_sumcheck_cluster" -c 3 -o $O/cfg2_cluster python tools/prof/cfg2_step.py > $O/ncu_cfg2c.log 2>&1; echo ncu_cfg2c rc=$?; tail -2 $O/ncu_cfg2c.log
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_mvt_rows|k_mvt_cols|k_mv_rows|k_mv_cols" -c 6 -o $O/cfg2_matvec python tools/prof/cfg2_step.py > $O/ncu_mv.log 2>&1; echo ncu_mv rc=$?; tail -2 $O/ncu_mv.log
ZKL_BENCH_OVERSUBSCRIBE=1 ZKL_NO_PERSISTENT=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_n2.json 2> $O/bench_n2.err; echo n2 rc=$?; tail -3 $O/bench_n2.err; python -c "import json; d=json.loads(open('$O/bench_n2.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['ms_per_step'], d['strong_scaling'])"
timeout 2700 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -6 $O/gpu_tests.log
