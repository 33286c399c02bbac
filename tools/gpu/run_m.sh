# r02: pipelined igemm16: block tests and block bench
set -x
O=gpurun_out/r02m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_witness.py tests/test_gpu_block.py -q -rA > $O/tests.log 2>&1; echo tests rc=$?; grep -E "passed|failed|FAILED|Error" $O/tests.log | head -20
timeout 1500 python bench.py --steps 10 --warmup 3 --no-cfg3 --no-cpu > $O/bench.json 2> $O/bench.err; echo bench rc=$?; tail -3 $O/bench.err
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); c=d['cfg4']; b=d['cfg5']['block_13b']; print(c['block_proof_s'], c['witness_s'], c['verifier_accept'], b['block_proof_s'], b['witness_s'], b['verifier_accept'])"
