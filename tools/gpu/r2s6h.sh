export PYTHONUNBUFFERED=1
for v in default yv default yv; do
  if [ $v = default ]; then unset HQ_LIB; else export HQ_LIB=tmp_variants/$v/libhoqri_b200.so; fi
  timeout 600 python tools/pass_time.py 2 2>&1 | grep -v Warn | tail -1
done
HQ_LIB=tmp_variants/yv/libhoqri_b200.so timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 600 2>&1 | tail -2
