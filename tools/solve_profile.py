"""One full BASELINE-config solve (all sweeps) for an ncu launch list: which kernels a real solve spends time in."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import CONFIGS, config_coo
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cid]
coords, vals = config_coo(cid)
dims, ranks = list(c["dims"]), list(c["ranks"])
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
x = hq.SparseTensor(dims, coords, vals)
u0 = hq.random_factors(dims, ranks, 1)
sol = hq.Solver(x, hq.SolverConfig(ranks=ranks, max_sweeps=c["sweeps"], tol_fit_change=0.0), init_factors=u0.factors,
                stream=s.cuda_stream)
sol.run(c["sweeps"]); sol.sync()
print(sol.status())
