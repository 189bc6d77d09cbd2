export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_skew.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do
timeout 300 python tools/pass_time.py 4 10 2>&1 | grep '^{'
HQ_LIB=$PWD/tmp_variants/novreg/libhoqri_b200.so timeout 300 python tools/pass_time.py 4 10 2>&1 | grep '^{'
done
HQ_LONG_SYNC=1 timeout 300 python tools/pass_time.py 3 10 2>&1 | grep '^{'
