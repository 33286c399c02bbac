# r02: block validity (tiny golden + reference verifiers in the loop, full-size witness range),
# parity at the stated configs, drop-in reference modules, cfg4 7B/13B block proof + verified proof
set -x
O=gpurun_out/r02b; mkdir -p $O
nproc; free -g | head -2
timeout 1800 python -m pytest tests/test_gpu_block.py -q -rA > $O/block_tests.log 2>&1; echo block rc=$?; grep -E "passed|failed|FAILED|Error" $O/block_tests.log | head -20
timeout 2400 python -m pytest tests/test_gpu_parity_scale.py -q -rA --durations=0 > $O/scale_tests.log 2>&1; echo scale rc=$?; grep -E "passed|failed|FAILED|Error|s call" $O/scale_tests.log | head -30
timeout 2400 python -m pytest tests/test_dropin_reference.py -q -rA > $O/dropin.log 2>&1; echo dropin rc=$?; grep -E "passed|failed|FAILED|Error" $O/dropin.log | head -30
timeout 1500 python bench.py --steps 10 --warmup 3 --no-cfg3 --no-cfg5 --no-cpu > $O/bench7.json 2> $O/bench7.err; echo b7 rc=$?; tail -3 $O/bench7.err
python -c "import json; d=json.loads(open('$O/bench7.json').read().strip().splitlines()[-1]); c=d['cfg4']; print(c['block_proof_s'], c['gadgets_per_block'], c['verify'])"
timeout 1500 python bench.py --steps 10 --warmup 3 --no-cfg3 --no-cfg5 --no-cpu --cfg4-shape 13b > $O/bench13.json 2> $O/bench13.err; echo b13 rc=$?; tail -3 $O/bench13.err
python -c "import json; d=json.loads(open('$O/bench13.json').read().strip().splitlines()[-1]); c=d['cfg4']; print(c['block_proof_s'], c['gadgets_per_block'], c['verify'])"
