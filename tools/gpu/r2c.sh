set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2c_ref.log 2>&1; echo "ref rc=$?"
tail -15 gpurun_out/r2c_pytest.log
tail -2 gpurun_out/r2c_bench.log
tail -2 gpurun_out/r2c_ref.log
