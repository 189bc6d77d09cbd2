export PYTHONUNBUFFERED=1
for i in 1 2; do
timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
HQ_LIB=$PWD/tmp_variants/nohint/libhoqri_b200.so timeout 300 python tools/pass_time.py 2 20 2>&1 | grep '^{'
done
timeout 300 python tools/timeline.py 2 5 2>&1 | grep -v -i warn | tail -11
