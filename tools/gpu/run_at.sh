# r02: ncu --set full of the new kernels: int64 tensor-core matvecs, GPU commitments, eq tree
O=gpurun_out/r02at; mkdir -p $O
python tools/prof/mv64_time.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mvt64 -c 4 -o $O/mvt64 python tools/prof/mv64_time.py > $O/ncu_mvt64.log 2>&1; echo mvt64 rc=$?
ncu --set full --clock-control none -k regex:k_q_commit_rows -c 2 -o $O/commit python tools/prof/commit_time.py > $O/ncu_commit.log 2>&1; echo commit rc=$?
ls -la $O
