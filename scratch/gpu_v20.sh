mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_v20.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest_v20.log
timeout 600 python bench.py > gpurun_out/bench_v20.json 2> gpurun_out/bench_v20.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_v20.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['value'], d['cfg3']['ms_per_proof'], d['cfg3']['sumcheck_ms_per_proof'], d['roofline']['frac'], d['cpu_baseline']['value'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_v20.json 2>&1; tail -1 gpurun_out/bench_ref_v20.json | cut -c1-300
