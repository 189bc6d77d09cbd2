export PYTHONUNBUFFERED=1
HQ_LIB=$PWD/tmp_variants/phase/libhoqri_b200.so timeout 300 python tools/phase_timing.py 2 > gpurun_out/r2f_phase.log 2>&1; echo "phase rc=$?"
cat gpurun_out/r2f_phase.log | tail -12
