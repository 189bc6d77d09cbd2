export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_qr_paths.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 600 2>&1 | tail -3
timeout 600 python tools/timeline.py 2 5 2>&1 | grep -v Warn | head -12
