# r02 first check: GPU tests (incl. the reference's own modules via install()), smoke
set -x
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -2 $O/smoke.log
timeout 2400 python -m pytest tests/test_dropin_reference.py -q -rA > $O/dropin.log 2>&1; echo dropin rc=$?; tail -15 $O/dropin.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_dropin_reference.py --deselect tests/test_gpu_block.py > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -5 $O/gpu_tests.log
