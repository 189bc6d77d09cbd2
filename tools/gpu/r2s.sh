export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_skew.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/pass_time.py 3 10 2>&1 | grep '^{'
HQ_LIB=$PWD/tmp_variants/ld3/libhoqri_b200.so timeout 300 python tools/pass_time.py 3 10 2>&1 | grep '^{'
timeout 600 python -m pytest tests/test_gpu_config_parity.py -q -s -p no:cacheprovider -k cfg3 2>&1 | grep "sweep\|passed\|failed"
