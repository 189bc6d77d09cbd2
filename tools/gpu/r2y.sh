export PYTHONUNBUFFERED=1
timeout 300 python tools/pass_time.py 3 10 2>&1 | grep '^{'
for v in smax64 smax128 smax512; do HQ_LIB=$PWD/tmp_variants/$v/libhoqri_b200.so timeout 300 python tools/pass_time.py 3 10 2>&1 | grep '^{'; done
