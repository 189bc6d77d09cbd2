export PYTHONUNBUFFERED=1
python tools/profile_pass.py 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pass_np3 -s 3 -c 1 -o gpurun_out/r2i_np3 python tools/profile_pass.py 2 > gpurun_out/r2i_ncu.log 2>&1; echo "ncu rc=$?"
HQ_LIB=$PWD/tmp_variants/base/libhoqri_b200.so ncu --set full --clock-control none --import-source on -k regex:k_pass_np3 -s 3 -c 1 -o gpurun_out/r2i_np3_base python tools/profile_pass.py 2 > gpurun_out/r2i_ncu_base.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/
