export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -rf --timeout 600 --deselect "tests/test_gpu_config_parity.py::test_config_trajectory_matches_reference[cfg2_s1.npz]" > gpurun_out/r2o_test.log 2>&1; echo "test rc=$?"; tail -8 gpurun_out/r2o_test.log
timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
timeout 300 python tools/timeline.py 2 5 2>&1 | tail -12
HQ_SEED=1 timeout 300 python tools/timeline.py 2 20 2>&1 | tail -14
