export PYTHONUNBUFFERED=1
for v in ku4 ku5 ku6 ku8 ku4; do
  export HQ_LIB=tmp_variants/$v/libhoqri_b200.so
  timeout 600 python tools/pass_time.py 2 2>&1 | grep -v Warn | tail -1
done
HQ_LIB=tmp_variants/ku4/libhoqri_b200.so timeout 600 python tools/pass_time.py 3 10 2>&1 | grep -v Warn | tail -1
