export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py tests/test_gpu_skew.py tests/test_gpu_dist1.py -q -x -p no:cacheprovider -rf > gpurun_out/r2j_test.log 2>&1; echo "test rc=$?"; tail -3 gpurun_out/r2j_test.log
timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
for v in pol1 pol2; do HQ_LIB=$PWD/tmp_variants/$v/libhoqri_b200.so timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'; done
timeout 300 python tools/pass_time.py 3 10 2>&1 | grep '^{'
HQ_LIB=$PWD/tmp_variants/phase/libhoqri_b200.so timeout 300 python tools/phase_timing.py 2 2>&1 | tail -10
