"""Which QR path each mode update takes on positive-valued (mean-dominated) data."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import uniform_coo
cases = [([20000] * 3, 200000, 10), ([50000] * 3, 500000, 10), ([100000] * 3, 1000000, 10), ([10000] * 3, 100000, 10),
         ([5000] * 3, 50000, 10)]
for dims, draws, k in cases:
    coords, vals = uniform_coo(dims, draws, 3)
    x = hq.SparseTensor(dims, coords, vals)
    u = hq.random_factors(dims, [k] * 3, 4)
    sol = hq.Solver(x, hq.SolverConfig(ranks=[k] * 3, max_sweeps=20, tol_fit_change=0.0), init_factors=u.factors)
    out = []
    t0 = time.perf_counter()
    for it in range(20):
        sol.run(1); sol.sync(); st = sol.status(); out.append((st["shifted"], st["fallbacks"]))
    print(dims, draws, f"{time.perf_counter() - t0:.3f}s", out, flush=True)
