export PYTHONUNBUFFERED=1
HQ_ITERS=10 HQ_PROFILE_BUILD=1 timeout 600 python tools/e2e_breakdown.py 2 2>&1 | grep -v "Warn\|status\|_warn" | tail -60
