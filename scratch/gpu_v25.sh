mkdir -p gpurun_out/v25
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py > gpurun_out/v25/bench.json 2> gpurun_out/v25/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/v25/bench.err
tail -1 gpurun_out/v25/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'], d['cfg3']['ms_per_proof'], d['lora_block_proof_s'], d['cfg5']['block_13b']['block_proof_s'], [ (r['n'], round(r['sumcheck_ms'],1), r['bit_exact_dense_vs_factored']) for r in d['cfg5']['sweep']], d['clocks'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_round -c 2 -o gpurun_out/v25/k_round_zkmat26 python scratch/sweep_ncu.py 26 > gpurun_out/v25/ncu1.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v25/sweep26_launches.csv python scratch/sweep_ncu.py 26 > /dev/null 2>&1; echo ncu2 rc=$?
python tools/ncu_launches.py gpurun_out/v25/sweep26_launches.csv | head -8
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_bench -c 1 -o gpurun_out/v25/mont_bench ./tools/mont_bench 2 200 > gpurun_out/v25/ncu3.log 2>&1; echo ncu3 rc=$?
