export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_qr_paths.py tests/test_gpu_parity.py tests/test_gpu_config_parity.py tests/test_gpu_dist1.py tests/test_gpu_dist2.py tests/test_gpu_dense.py -m gpu -q -x -p no:cacheprovider --timeout 600 2>&1 | tail -3
timeout 600 python tools/timeline.py 2 5 x 2>&1 | grep -v Warn | grep -A16 "launch sequence"
timeout 600 python tools/pass_time.py 2 2>&1 | grep -v Warn | tail -1
timeout 600 python tools/pass_time.py 4 2>&1 | grep -v Warn | tail -1
