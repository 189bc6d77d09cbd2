export PYTHONUNBUFFERED=1
HQ_LIB=tmp_variants/alloct/libhoqri_b200.so HQ_ITERS=14 timeout 600 python tools/e2e_breakdown.py 2 2>&1 | grep "tensor=" | tail -60
python - <<'P'
import paper_2510_16930_b200 as hq
print("freed", hq.release_cached_memory())
P
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 600 2>&1 | tail -3
