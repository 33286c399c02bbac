# r02: replay-mode debug, sharded proving (multi-process on one GPU), the full GPU suite
set -x
O=gpurun_out/r02d; mkdir -p $O
ZKL_PROFILE_REPLAY=1 timeout 600 python tools/prof/replay_dbg.py > $O/replay_dbg.log 2>&1; echo replay rc=$?; cat $O/replay_dbg.log | tail -8
timeout 1800 python -m pytest tests/test_gpu_shard.py -q -rA > $O/shard_tests.log 2>&1; echo shard rc=$?; grep -E "passed|failed|FAILED|Error" $O/shard_tests.log | head -20
timeout 2700 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_parity.py::test_profile_replay_mode_matches_oracle --deselect tests/test_gpu_shard.py > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -8 $O/gpu_tests.log
for k in k_range_count16 k_rescale_witness k_lift16_lut; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $O/hbm_$k python tools/prof/block_lookup.py > $O/ncu_$k.log 2>&1; echo ncu $k rc=$?
done
