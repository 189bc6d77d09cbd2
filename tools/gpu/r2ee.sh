export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_fast.py tests/test_gpu_skew.py -q -x -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do for c in 2 3; do
timeout 300 python tools/pass_time.py $c 10 2>&1 | grep '^{'
HQ_LIB=$PWD/tmp_variants/base2/libhoqri_b200.so timeout 300 python tools/pass_time.py $c 10 2>&1 | grep '^{'
done; done
