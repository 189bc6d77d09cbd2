export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass_np3 --launch-skip 7 --launch-count 2 -o gpurun_out/s3d_pass python tools/profile_sweep.py 2 > gpurun_out/s3d_ncu.log 2>&1; echo rc=$?
