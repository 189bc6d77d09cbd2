export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 600 > gpurun_out/r2m_test.log 2>&1; echo "test rc=$?"; tail -8 gpurun_out/r2m_test.log
timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
timeout 300 python tools/timeline.py 2 5 2>&1 | tail -12
