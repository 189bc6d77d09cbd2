export PYTHONUNBUFFERED=1
HQ_LIB=$PWD/tmp_variants/pt/libhoqri_b200.so timeout 600 python tools/fib_phase_timing.py 3 2>&1 | tail -32
