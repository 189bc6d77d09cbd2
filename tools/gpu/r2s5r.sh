export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 600 > $O/s5r_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/s5r_pytest.log
timeout 900 python bench.py > $O/s5r_bench2.log 2>&1; echo "bench2 rc=$?"; tail -c 300 $O/s5r_bench2.log
for c in 3 4 5; do timeout 900 python bench.py --config $c --no-cpu > $O/s5r_bench$c.log 2>&1; echo "bench$c rc=$?"; done
python -c "import __graft_entry__ as g; g.smoke()" > $O/s5r_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/s5r_smoke.log
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > $O/s5r_bench2_g2.log 2>&1; echo "bench --gpus 2 rc=$?"; tail -c 1200 $O/s5r_bench2_g2.log
