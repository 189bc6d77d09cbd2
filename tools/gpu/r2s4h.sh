export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_skew.py -q -p no:cacheprovider -x --timeout 600 2>&1 | tail -3
for v in default cap8 cap4; do
  if [ $v != default ]; then export HQ_LIB=$PWD/tmp_variants/$v/libhoqri_b200.so; fi
  echo "== $v"
  timeout 600 python tools/timeline.py 3 5 seq 2>&1 | grep -v Warn | grep -E "span|fibseg|np3" | head -8
done
HQ_LIB=$PWD/tmp_variants/pt4/libhoqri_b200.so timeout 600 python tools/fib_phase_timing.py 3 2>&1 | tail -27 | head -18
HQ_LIB=$PWD/tmp_variants/cap4/libhoqri_b200.so timeout 900 python -m pytest tests/test_gpu_skew.py -q -p no:cacheprovider --timeout 600 2>&1 | tail -3
