export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 600 > gpurun_out/s4k_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/s4k_pytest.log
for c in 3 2 4; do
timeout 600 python tools/timeline.py $c 5 2>&1 | grep -v Warn | head -9
done
timeout 600 python bench.py --config 3 --no-cpu > gpurun_out/s4k_bench3.log 2>&1; echo "bench3 rc=$?"; tail -c 1500 gpurun_out/s4k_bench3.log
