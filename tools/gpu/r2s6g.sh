export PYTHONUNBUFFERED=1
timeout 600 python tools/pass_time.py 2 2>&1 | grep -v Warn | tail -1
timeout 1200 python -m pytest tests/test_gpu_fast.py tests/test_gpu_skew.py tests/test_gpu_parity.py tests/test_gpu_config_parity.py -m gpu -q -x -p no:cacheprovider --timeout 600 2>&1 | tail -2
