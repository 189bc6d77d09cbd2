export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_qr_paths.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
timeout 300 python tools/timeline.py 2 5 2>&1 | grep -v -i warn | tail -11
