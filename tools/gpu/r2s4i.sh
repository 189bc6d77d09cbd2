export PYTHONUNBUFFERED=1
for v in default dv un sm128 sm64; do
  if [ $v != default ]; then export HQ_LIB=$PWD/tmp_variants/$v/libhoqri_b200.so; fi
  echo "== $v"
  timeout 600 python tools/timeline.py 3 5 seq 2>&1 | grep -v Warn | grep -E "span|fibseg|np3|longfix" | head -9
done
