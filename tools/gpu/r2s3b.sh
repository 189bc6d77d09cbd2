export PYTHONUNBUFFERED=1
timeout 300 python tools/timeline.py 2 5 seq > gpurun_out/s3b_tl2.log 2>&1; echo rc=$?
timeout 300 python tools/timeline.py 3 3 seq > gpurun_out/s3b_tl3.log 2>&1; echo rc=$?
head -30 gpurun_out/s3b_tl2.log
