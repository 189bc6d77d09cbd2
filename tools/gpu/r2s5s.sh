export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 2 > $O/s5s_bench2.log 2>&1; echo "bench2 rc=$?"; tail -c 400 $O/s5s_bench2.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 600 > $O/s5s_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/s5s_pytest.log
