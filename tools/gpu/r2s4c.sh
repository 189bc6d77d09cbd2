export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_skew.py -q -p no:cacheprovider -x --timeout 600 2>&1 | tail -15
echo "== config 3 fibers auto"
timeout 600 python tools/timeline.py 3 5 2>&1 | grep -v Warn | head -16
echo "== config 3 fibers off"
HQ_FIBERS=0 timeout 600 python tools/timeline.py 3 5 2>&1 | grep -v Warn | head -8
