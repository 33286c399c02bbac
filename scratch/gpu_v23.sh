mkdir -p gpurun_out/v23
timeout 600 python scratch/block_prof.py > gpurun_out/v23/block_prof.log 2>&1; echo "rc=$?"; head -80 gpurun_out/v23/block_prof.log
timeout 600 python scratch/block_prof.py stages > gpurun_out/v23/block_prof_stages.log 2>&1; echo "rc=$?"; grep -A30 -- "--- stages" gpurun_out/v23/block_prof_stages.log; head -1 gpurun_out/v23/block_prof_stages.log
