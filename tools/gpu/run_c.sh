# r02: full GPU suite, ncu of the production round kernels (recorded-challenge replay) and
# of the HBM-bound block passes, launch list of the cfg2 step, default bench
set -x
O=gpurun_out/r02c; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf -x > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -8 $O/gpu_tests.log
timeout 900 env ZKL_PROFILE_REPLAY=1 ncu --set full --import-source on --clock-control none -k regex:"k_sumcheck_(persistent|cluster)" -c 2 -o $O/dense26_full python tools/prof/sweep_point.py 26 > $O/ncu_dense.log 2>&1; echo ncu_dense rc=$?; tail -3 $O/ncu_dense.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_range_count16|k_rescale_witness|k_lift16" -c 3 -o $O/hbm_full python tools/prof/block_lookup.py > $O/ncu_hbm.log 2>&1; echo ncu_hbm rc=$?; tail -3 $O/ncu_hbm.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg2.csv python tools/prof/cfg2_step.py > $O/ncu_cfg2.log 2>&1; echo ncu_cfg2 rc=$?
python tools/ncu_launches.py $O/launches_cfg2.csv > $O/launches_cfg2.summary.txt 2>&1; head -20 $O/launches_cfg2.summary.txt
timeout 1800 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?; tail -3 $O/bench.err
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['cpu_baseline'] and {k: d['cpu_baseline'][k] for k in ('value','kind')}, d['cfg3']['ms_per_proof'], d['lora_block_proof_s'], d['cfg4']['verifier_accept'], d['cfg5']['block_13b']['block_proof_s'], d['cfg5']['block_13b']['verifier_accept'], d['clocks'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2>&1; echo ref rc=$?; tail -c 400 $O/bench_ref.json
