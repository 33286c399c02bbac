# r02: large witness products through the library int8 GEMM
O=gpurun_out/r02ak; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_witness.py tests/test_gpu_block.py -q -x > $O/tests.log 2>&1; echo tests rc=$?; tail -2 $O/tests.log
python tools/prof/igemm_time.py > $O/igemm.jsonl 2>&1; cat $O/igemm.jsonl | cut -c1-150
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench.json 2> $O/bench.err; echo bench rc=$?; tail -3 $O/bench.err
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['operands_copied']['ms_per_step'])"
timeout 900 python tools/prof/witness_time.py > $O/witness.jsonl 2>&1; cut -c1-200 $O/witness.jsonl
