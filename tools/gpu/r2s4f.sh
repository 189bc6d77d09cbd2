export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fibseg --launch-skip 6 --launch-count 3 -o gpurun_out/s4f_fibseg python tools/profile_sweep.py 3 > gpurun_out/s4f_ncu.log 2>&1; echo rc=$?
tail -3 gpurun_out/s4f_ncu.log
