export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_qr_paths.py tests/test_gpu_config_parity.py tests/test_gpu_dist2.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 600 2>&1 | tail -3
timeout 300 python tools/hh_time.py 2>&1 | grep -v Warn | tail -5
