export PYTHONUNBUFFERED=1
HQ_LIB=tmp_variants/phase/libhoqri_b200.so timeout 600 python tools/phase_timing.py 2 2>&1 | grep -v Warn
timeout 600 python tools/pass_time.py 2 2>&1 | grep -v Warn | tail -8
