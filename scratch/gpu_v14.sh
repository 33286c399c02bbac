./tools/mont_bench 2 2000 | head -3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_v14.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest_v14.log
python scratch/cfg3_prof.py 2>&1 | head -4
timeout 600 python bench.py > gpurun_out/bench_v14.json 2> gpurun_out/bench_v14.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_v14.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['value'], d['cfg3']['ms_per_proof'], d['cfg3']['sumcheck_ms_per_proof'], d['round_engine'] if 'round_engine' in d else '')"
