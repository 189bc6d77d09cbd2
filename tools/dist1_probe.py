import sys; sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import config_coo
coords, vals = config_coo(2)
dims, k = [1000000] * 3, 10
x = hq.SparseTensor(dims, coords, vals)
u = hq.random_factors(dims, [k] * 3, 1).factors
for comm in (None, hq.Comm(1, 0)):
    sol = hq.Solver(x, hq.SolverConfig(ranks=[k]*3, max_sweeps=20, tol_fit_change=0.0), init_factors=u, comm=comm)
    out = []
    for i in range(20):
        sol.run(1)
        try:
            sol.sync()
        except Exception as e:
            out.append(("EXC", str(e)[:60])); break
        st = sol.status(); out.append((st["sweeps"], st["shifted"], st["fallbacks"], st["deficient_kept"], st["abort"]))
    print("dist" if comm else "single", out, flush=True)
