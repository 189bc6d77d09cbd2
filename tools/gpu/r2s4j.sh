export PYTHONUNBUFFERED=1
for v in sm48 sm32 sm16; do
  export HQ_LIB=$PWD/tmp_variants/$v/libhoqri_b200.so
  echo "== $v"
  timeout 600 python tools/timeline.py 3 5 seq 2>&1 | grep -v Warn | grep -E "span|fibseg|np3|longfix" | head -7
done
