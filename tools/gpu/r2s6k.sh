export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 600 > $O/s6k_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/s6k_pytest.log
for c in 3 4 5; do timeout 900 python bench.py --config $c --no-cpu > $O/s6k_bench$c.log 2>&1; echo "bench$c rc=$?"; done
