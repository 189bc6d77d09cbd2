export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_skew.py tests/test_gpu_parity.py tests/test_gpu_dist1.py tests/test_gpu_dist2.py -q -x -p no:cacheprovider 2>&1 | tail -3
for c in 2 3; do
timeout 300 python tools/pass_time.py $c 10 2>&1 | grep '^{'
HQ_LIB=$PWD/tmp_variants/base2/libhoqri_b200.so timeout 300 python tools/pass_time.py $c 10 2>&1 | grep '^{'
done
timeout 600 python -m pytest tests/test_gpu_config_parity.py -q -s -p no:cacheprovider -k "cfg3 or cfg2_s2025" 2>&1 | grep "sweep\|passed\|failed" | head -30
