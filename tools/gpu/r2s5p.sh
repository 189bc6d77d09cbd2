export PYTHONUNBUFFERED=1
for v in cholrt cholct cholrt cholct; do
HQ_LIB=tmp_variants/$v/libhoqri_b200.so timeout 600 python tools/timeline.py 2 10 2>&1 | grep "k_chol\|span" | sed "s/^/$v /"
done
