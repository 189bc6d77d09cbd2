export PYTHONUNBUFFERED=1
for i in 1 2; do
timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
HQ_LIB=$PWD/tmp_variants/fw22/libhoqri_b200.so timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
done
HQ_LIB=$PWD/tmp_variants/fw22/libhoqri_b200.so timeout 300 python tools/pass_time.py 3 10 2>&1 | grep '^{'
