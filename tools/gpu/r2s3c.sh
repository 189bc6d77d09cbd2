export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_chol1|k_chol2|k_reduce_pass|k_gt|k_rowgemm_tma" --launch-skip 40 --launch-count 12 -o gpurun_out/s3c_small python tools/profile_sweep.py 2 > gpurun_out/s3c_ncu.log 2>&1; echo rc=$?
tail -3 gpurun_out/s3c_ncu.log
