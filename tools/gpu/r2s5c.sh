export PYTHONUNBUFFERED=1
timeout 600 python tools/e2e_breakdown.py 2 2>&1 | grep -v Warn | grep -v status
