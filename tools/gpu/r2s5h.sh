export PYTHONUNBUFFERED=1
timeout 600 python tools/timeline.py 2 5 x 2>&1 | grep -v Warn | sed -n 1,6p
timeout 600 python tools/timeline.py 2 5 x 2>&1 | grep -A16 "launch sequence"
HQ_NO_REVERSE=1 timeout 600 python tools/timeline.py 2 5 x 2>&1 | grep -A16 "launch sequence"
