export PYTHONUNBUFFERED=1
HQ_ITERS=12 HQ_PROFILE_BUILD=1 timeout 600 python tools/e2e_breakdown.py 2 2>&1 | grep "sort buffers\|radix sort\|lexsort\|upload wait\|tensor=" | tail -60
