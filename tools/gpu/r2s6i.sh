export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 900 python bench.py > $O/s6i_bench2.log 2>&1; echo "bench2 rc=$?"; tail -c 300 $O/s6i_bench2.log
for c in 3 4 5; do timeout 900 python bench.py --config $c --no-cpu > $O/s6i_bench$c.log 2>&1; echo "bench$c rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/s6i_launches_bench2.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $O/s6i_ncu_bench2.log 2>&1; echo "ncu-list2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_np3 --launch-skip 8 --launch-count 2 -o $O/s6i_np3 -f python tools/profile_sweep.py 2 > $O/s6i_ncu_np3.log 2>&1; echo "ncu-np3 rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 600 > $O/s6i_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/s6i_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/s6i_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/s6i_smoke.log
