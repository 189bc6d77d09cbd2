set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_dist2.py tests/test_gpu_skew.py -q -p no:cacheprovider -rf > gpurun_out/r2e_dist.log 2>&1; echo "dist rc=$?"
HQ_LIB=$PWD/tmp_variants/noshift/libhoqri_b200.so timeout 1800 python -m pytest tests/test_gpu_config_parity.py -q -s -p no:cacheprovider -rf > gpurun_out/r2e_cfg_noshift.log 2>&1; echo "cfg rc=$?"
timeout 1800 python -m pytest tests/test_gpu_config_parity.py -q -s -p no:cacheprovider -rf > gpurun_out/r2e_cfg.log 2>&1; echo "cfg rc=$?"
tail -3 gpurun_out/r2e_dist.log
grep -n "sweep\|status\|passed\|failed" gpurun_out/r2e_cfg_noshift.log | head -80
