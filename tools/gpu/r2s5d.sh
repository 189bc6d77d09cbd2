export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_skew.py -m gpu -q -x -p no:cacheprovider --timeout 600 2>&1 | tail -3
for v in default gtl nopf; do
  if [ $v = default ]; then unset HQ_LIB; else export HQ_LIB=tmp_variants/$v/libhoqri_b200.so; fi
  timeout 600 python tools/pass_time.py 2 2>&1 | grep -v Warn | tail -1
done
HQ_LIB=tmp_variants/phase/libhoqri_b200.so timeout 600 python tools/phase_timing.py 2 2>&1 | grep -v Warn
unset HQ_LIB
timeout 600 python tools/pass_time.py 3 2>&1 | grep -v Warn | tail -1
