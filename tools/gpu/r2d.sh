set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_dist2.py tests/test_gpu_skew.py -q -p no:cacheprovider -rf -x > gpurun_out/r2d_dist.log 2>&1; echo "dist rc=$?"
for v in base; do HQ_LIB=$PWD/tmp_variants/$v/libhoqri_b200.so timeout 300 python tools/pass_time.py 2 20 >> gpurun_out/r2d_pt.log 2>&1; done
timeout 300 python tools/pass_time.py 2 20 >> gpurun_out/r2d_pt.log 2>&1
HQ_LIB=$PWD/tmp_variants/base/libhoqri_b200.so timeout 300 python tools/pass_time.py 3 10 >> gpurun_out/r2d_pt.log 2>&1
timeout 300 python tools/pass_time.py 3 10 >> gpurun_out/r2d_pt.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_config_parity.py -q -s -p no:cacheprovider -rf > gpurun_out/r2d_cfg.log 2>&1; echo "cfg rc=$?"
tail -5 gpurun_out/r2d_dist.log; cat gpurun_out/r2d_pt.log | grep '^{'
grep -n "sweep\|status\|passed\|failed" gpurun_out/r2d_cfg.log | head -80
