export PYTHONUNBUFFERED=1
for v in default fibu fibd0 default; do
  if [ $v = default ]; then unset HQ_LIB; else export HQ_LIB=tmp_variants/$v/libhoqri_b200.so; fi
  timeout 600 python tools/pass_time.py 3 8 2>&1 | grep -v Warn | tail -1
done
