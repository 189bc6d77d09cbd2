export PYTHONUNBUFFERED=1
timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
for v in w2mb5 w2mb4; do HQ_LIB=$PWD/tmp_variants/$v/libhoqri_b200.so timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'; done
HQ_LIB=$PWD/tmp_variants/w2mb5/libhoqri_b200.so timeout 600 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_config_parity.py -q -p no:cacheprovider -k "cfg2_s1" 2>&1 | tail -2
