export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_skew.py -q -p no:cacheprovider -x --timeout 600 2>&1 | tail -15
for c in 4 3 2; do
echo "== config 3 fused, CTAs/SM <= $c"
HQ_FIB_CTAS=$c timeout 600 python tools/timeline.py 3 5 seq 2>&1 | grep -v Warn | grep -E "span|fibseg|np3|longfix" | head -12
done
