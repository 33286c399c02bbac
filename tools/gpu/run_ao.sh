# r02: eq point staged in device memory; four-lane vs one-lane tree
for v in default eq1; do
  if [ $v = eq1 ]; then export ZKL_LIB=build/variants/eq1/libzkl_b200.so; else unset ZKL_LIB; fi
  python tools/prof/cfg2_timeline.py gpurun_out/timeline_$v > /dev/null 2>&1
  echo "$v eq: $(grep eq_tree gpurun_out/timeline_$v/cfg2_timeline.txt | awk '{s+=$2; n++} END {print n, s}') $(grep point_to_dev gpurun_out/timeline_$v/cfg2_timeline.txt | awk '{s+=$2; n++} END {print n, s}') $(tail -1 gpurun_out/timeline_$v/cfg2_timeline.txt)"
  timeout 900 python bench.py --steps 20 --warmup 3 --no-cfg3 --no-cfg4 --no-cfg5 --no-cpu > gpurun_out/bench_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "eq or matmul or golden" 2>&1 | tail -1
