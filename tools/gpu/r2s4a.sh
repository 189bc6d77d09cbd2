export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4a_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4a_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 600 > gpurun_out/s4a_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4a_pytest.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4a_bench.log 2>&1; echo "bench rc=$?"
timeout 300 python tools/timeline.py 2 5 seq > gpurun_out/s4a_timeline2.log 2>&1; echo "tl2 rc=$?"
timeout 300 python tools/timeline.py 3 5 seq > gpurun_out/s4a_timeline3.log 2>&1; echo "tl3 rc=$?"
tail -c 600 gpurun_out/s4a_bench.log; echo
head -30 gpurun_out/s4a_timeline2.log
