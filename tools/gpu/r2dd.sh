export PYTHONUNBUFFERED=1
for c in 2 3; do
timeout 300 python tools/pass_time.py $c 10 2>&1 | grep '^{'
HQ_LIB=$PWD/tmp_variants/noorder/libhoqri_b200.so timeout 300 python tools/pass_time.py $c 10 2>&1 | grep '^{'
HQ_LIB=$PWD/tmp_variants/tc0/libhoqri_b200.so timeout 300 python tools/pass_time.py $c 10 2>&1 | grep '^{'
done
