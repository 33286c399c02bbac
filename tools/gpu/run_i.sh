# r02: sharded engine (persistent path in a one-rank group; lookups sharded from 4 ranks)
set -x
O=gpurun_out/r02i; mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_shard.py -q -rA > $O/shard_tests.log 2>&1; echo shard rc=$?; grep -E "passed|failed|FAILED|Error" $O/shard_tests.log | head -20
