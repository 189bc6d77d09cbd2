import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import uniform_coo
for dims, draws in [([2000,1500,1000], 50000), ([100000]*3, 1000000)]:
    coords, vals = uniform_coo(dims, draws, 3)
    x = hq.SparseTensor(dims, coords, vals)
    u = hq.random_factors(dims, [10]*3, 4)
    for ms in (6, 20):
        sol = hq.Solver(x, hq.SolverConfig(ranks=[10]*3, max_sweeps=ms, tol_fit_change=0.0), init_factors=u.factors)
        sol.run(1); sol.sync(); a = sol.status()
        sol.run(2); sol.sync(); b = sol.status()
        sol.run(ms-3); sol.sync(); c = sol.status()
        print(dims, ms, a, b, c, flush=True)
