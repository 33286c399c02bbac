# r02: matvec finish fused into the tensor-core kernels (last CTA per output tile)
O=gpurun_out/r02bd; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_witness.py tests/test_gpu_commit.py -q -x > $O/tests.log 2>&1; echo tests rc=$?; tail -1 $O/tests.log
for i in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > $O/bench_$i.json 2> $O/bench_$i.err; echo bench rc=$?
python -c "import json; d=json.loads(open('$O/bench_$i.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel_only'])"
done
python tools/prof/cfg2_timeline.py > $O/timeline.log 2>&1; cp gpurun_out/timeline/cfg2_timeline.txt $O/
