set -x
python -m pytest tests/test_gpu_config_parity.py -x -q -s > gpurun_out/r2b_cfgpar.log 2>&1; echo "cfgpar rc=$?"
python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/r2b_fast.log 2>&1; echo "fast rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b_ref.log 2>&1; echo "ref rc=$?"
tail -5 gpurun_out/r2b_cfgpar.log
