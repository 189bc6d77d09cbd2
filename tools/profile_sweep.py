"""Runs a few HOQRI sweeps of BASELINE config 2 through the device solver (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import CONFIGS, config_coo
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cfg_id]
coords, vals = config_coo(cfg_id)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
x = hq.SparseTensor(list(c["dims"]), coords, vals)
u0 = hq.random_factors(list(c["dims"]), list(c["ranks"]), 1)
sol = hq.Solver(x, hq.SolverConfig(ranks=list(c["ranks"]), max_sweeps=6, tol_fit_change=0.0), init_factors=u0.factors,
                stream=s.cuda_stream)
sol.run(4); sol.sync()
torch.cuda.synchronize()
print("ok")
