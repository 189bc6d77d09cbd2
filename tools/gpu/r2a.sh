set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.log 2>&1; echo "bench rc=$?"
python tools/profile_pass.py 2 > gpurun_out/r2a_pp.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pass_np3 -s 3 -c 1 -o gpurun_out/r2a_np3 python tools/profile_pass.py 2 > gpurun_out/r2a_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r2a_pytest.log
