set -x
mkdir -p gpurun_out/r02l
python -m pytest tests/test_gpu_witness.py -x -q 2>&1 | tail -5 > gpurun_out/r02l/witness_tests.log
python tools/prof/igemm_time.py > gpurun_out/r02l/igemm_time.jsonl 2>&1
cat gpurun_out/r02l/witness_tests.log gpurun_out/r02l/igemm_time.jsonl
