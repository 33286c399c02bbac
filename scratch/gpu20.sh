mkdir -p gpurun_out/p7
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/p7/launches.csv python scratch/prof_step.py > /dev/null 2>&1; echo ncu1 rc=$?
python tools/ncu_launches.py gpurun_out/p7/launches.csv > gpurun_out/p7/launches.summary.txt; head -16 gpurun_out/p7/launches.summary.txt
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_round -c 1 -o gpurun_out/p7/k_round python scratch/prof_step.py > /dev/null 2>&1; echo ncu4 rc=$?
timeout 120 compute-sanitizer --tool memcheck python -c "
import sys; sys.path[:0]=['.','tests','tests/golden']
import test_gpu_parity as T
T.test_matmul_factored_vs_oracle('big', (5, 9, 3), 'i16', 'native')
T.test_sumcheck_shapes_vs_oracle('big', 6, 'sum2prod2')
print('sanitizer run ok')" 2>&1 | tail -4
