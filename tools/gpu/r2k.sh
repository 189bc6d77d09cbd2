export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -rf > gpurun_out/r2k_test.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/r2k_test.log
timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
for v in nq1 nq2 nq8; do HQ_LIB=$PWD/tmp_variants/$v/libhoqri_b200.so timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'; done
