export PYTHONUNBUFFERED=1
V=$PWD/tmp_variants/pipe/libhoqri_b200.so
timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
HQ_LIB=$V timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
HQ_LIB=$V timeout 300 python tools/pass_time.py 3 10 2>&1 | grep '^{'
HQ_LIB=$PWD/tmp_variants/pipeph/libhoqri_b200.so timeout 200 python tools/phase_pipe.py 2 2>&1 | grep -v Warn
HQ_LIB=$V timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py tests/test_gpu_skew.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
