export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 600 > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2r_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2r_bench2.log 2>&1; echo "bench rc=$?"
for c in 3 4 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/r2r_bench$c.log 2>&1; echo "bench$c rc=$?"; done
python tools/profile_pass.py 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pass_np3 -s 3 -c 1 -o gpurun_out/r2r_np3 python tools/profile_pass.py 2 > gpurun_out/r2r_ncu.log 2>&1; echo "ncu rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2r_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1; echo "launches rc=$?"
tail -c 1500 gpurun_out/r2r_bench2.log
