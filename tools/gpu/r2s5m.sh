export PYTHONUNBUFFERED=1
HQ_LIB=tmp_variants/alloct/libhoqri_b200.so HQ_ITERS=14 timeout 600 python tools/e2e_breakdown.py 2 2>&1 | grep "alloc\]\|free\]\|tensor=" | tail -60
