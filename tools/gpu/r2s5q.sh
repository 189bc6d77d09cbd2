export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_dist2.py tests/test_gpu_dist1.py -m gpu -q -x -p no:cacheprovider --timeout 600 2>&1 | tail -30
