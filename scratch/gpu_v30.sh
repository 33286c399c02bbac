mkdir -p gpurun_out/v30
python scratch/hbm_ncu.py
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_lift|k_rescale_witness|k_range_count" -c 3 -o gpurun_out/v30/hbm_kernels python scratch/hbm_ncu.py > gpurun_out/v30/ncu.log 2>&1; echo ncu rc=$?
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
