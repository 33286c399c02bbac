mkdir -p gpurun_out/v29
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v29/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/v29/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/v29/bench.json 2> gpurun_out/v29/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/v29/bench.err
tail -1 gpurun_out/v29/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['cfg3']['ms_per_proof'], d['lora_block_proof_s'], d['cfg5']['block_13b']['block_proof_s'], [ (r['n'], round(r['sumcheck_ms'],1), r['bit_exact_dense_vs_factored']) for r in d['cfg5']['sweep']], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/v29/bench_reference.json 2>&1; tail -1 gpurun_out/v29/bench_reference.json | cut -c1-200
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
