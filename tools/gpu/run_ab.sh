# r02: debug graph path
O=gpurun_out/r02ab; mkdir -p $O
ZKL_NO_GRAPHS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "test_prove_matmul_full_with_stub_openings" > $O/t1.log 2>&1; echo nographs rc=$?; tail -1 $O/t1.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "test_prove_matmul_full_with_stub_openings" > $O/t2.log 2>&1; echo graphs-alone rc=$?; tail -1 $O/t2.log
timeout 600 python tools/prof/graph_dbg.py > $O/dbg.log 2>&1; echo dbg rc=$?; tail -30 $O/dbg.log
