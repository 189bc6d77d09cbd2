export PYTHONUNBUFFERED=1
cat > /tmp/small.py <<'P'
import numpy as np, sys
sys.path.insert(0,'.')
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import uniform_coo, zipf_coo
for dims, n, k, gen in (([3000,2500,2000], 60000, 10, 'u'), ([400,300,200], 200000, 10, 'z'), ([500,400,300], 150000, 16, 'u'), ([60,50,40,30], 100000, 8, 'u')):
    coords, vals = (uniform_coo(dims, n, 3) if gen == 'u' else zipf_coo(dims, n, 3))
    x = hq.SparseTensor(dims, coords, vals)
    r = hq.hoqri(x, hq.SolverConfig(ranks=[k]*len(dims), max_sweeps=3, tol_fit_change=0.0))
    print(dims, k, r.trace.sweeps[-1].objective)
print("freed", hq.release_cached_memory())
P
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 7 python /tmp/small.py 2>&1 | tail -12; echo "memcheck rc=${PIPESTATUS[0]}"
