export PYTHONUNBUFFERED=1
for v in default rec128 rec256 default rec256; do
  if [ $v = default ]; then unset HQ_LIB; else export HQ_LIB=tmp_variants/$v/libhoqri_b200.so; fi
  timeout 600 python tools/pass_time.py 2 2>&1 | grep -v Warn | tail -1
done
