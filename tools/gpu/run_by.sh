# r02: final validation (fused pair poll + tail)
set -x
O=gpurun_out/r02by; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 2700 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -4 $O/gpu_tests.log
timeout 1800 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?; tail -3 $O/bench.err
python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1])
c=d['cpu_baseline']
print('cfg2', d['ms_per_step'], d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['roofline']['traffic'], d['round_engine']['us_per_round'], d['clocks'])
print('cpu', c['value'], c['kind'], c['factored_port']['value'], c['factored_port']['seconds_per_step'], c.get('cfg3_reference', {}).get('extrapolated_seconds_per_proof'), c.get('commitment_reference', {}).get('s_per_entry'))
print('cfg3', d['cfg3']['ms_per_proof'])
print('cfg4', d['cfg4']['block_proof_s'], d['cfg4']['verifier_accept'], d['cfg4']['gadgets_per_block'], d['cfg4']['rounds_per_block'])
b=d['cfg5']['block_13b']; print('13b', b['block_proof_s'], b['verifier_accept'], b['gadgets_per_block'], b['rounds_per_block'])
print('sweep', [(r['n'], round(r['sumcheck_ms'],1), r['bit_exact_dense_vs_factored']) for r in d['cfg5']['sweep']])
print('hbm', {k: round(v['frac'],3) for k,v in d['hbm_kernels']['kernels'].items()})
"
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2>&1; echo ref rc=$?; tail -c 300 $O/bench_ref.json
